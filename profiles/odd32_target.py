"""ncu target: stream-major fills of xoshiro128** (u32) with aligned rows
(T = 1024, TMA) and odd rows (T = 1023, row-group TMA), 2^21 substreams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec(sys.argv[1] if len(sys.argv) > 1 else "xoshiro128starstar")
n = 1 << 21
sub = D.Substreams.from_seed(spec, 7, n)
for T in (1024, 1023):
    out = torch.empty((n, T), dtype=torch.uint32, device="cuda")
    for _ in range(2):
        D.fill(spec, sub.states, T, out=out)
    torch.cuda.synchronize()
    del out
print("ok")

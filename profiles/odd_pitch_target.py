"""ncu target: one stream-major fill of xoshiro256** with an aligned row
(T = 2048, TMA) and an odd row (T = 2047, row-group TMA), 2^19 substreams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec("xoshiro256starstar")
n = 1 << 19
sub = D.Substreams.from_seed(spec, 42, n)
for T in (2048, 2047):
    out = torch.empty((n, T), dtype=torch.uint64, device="cuda")
    for _ in range(2):
        D.fill(spec, sub.states, T, out=out)
    torch.cuda.synchronize()
    del out

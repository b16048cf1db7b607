"""ncu target: one position-major fill with an odd pitch (FILL_POS direct
stores) and the same shape aligned (TMA), xoshiro256**, 2^20 (+1) x 1024."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec("xoshiro256starstar")
for n in ((1 << 20) + 1, 1 << 20):
    sub = D.Substreams.from_seed(spec, 42, n)
    out = torch.empty((1024, n), dtype=torch.uint64, device="cuda")
    for _ in range(2):
        sub.fill(1024, out=out, layout="position")
torch.cuda.synchronize()
print("ok")

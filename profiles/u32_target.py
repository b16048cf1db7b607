"""ncu target: config-4 store fill, xoshiro128** u32 and f32, 2^22 x 1024."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec(sys.argv[1] if len(sys.argv) > 1 else "xoshiro128starstar")
n, T = 1 << 22, 1024
sub = D.Substreams.from_seed(spec, 7, n)
out = torch.empty((n, T), dtype=torch.uint32, device="cuda")
outf = torch.empty((n, T), dtype=torch.float32, device="cuda")
for _ in range(2):
    sub.fill(T, out=out)
    sub.fill(T, out=outf, kind="f32")
torch.cuda.synchronize()
print("ok")

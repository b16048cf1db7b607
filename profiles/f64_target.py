"""ncu target: config-2 store of xoshiro256** converted to float64 (K3
epilogue of k_fill), 2^20 x 1024, after one warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec(sys.argv[1] if len(sys.argv) > 1 else "xoshiro256starstar")
n, T = 1 << 20, 1024
sub = D.Substreams.from_seed(spec, 42, n)
out = torch.empty((n, T), dtype=torch.float64, device="cuda")
for _ in range(2):
    sub.fill(T, out=out, kind="f64")
torch.cuda.synchronize()
print("ok")

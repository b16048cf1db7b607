"""Short, fixed workload for ncu captures (one GPU): config-2 substream init
(K1), one store fill (K2, TMA) and one fused checksum (K4) for xoshiro256**,
after one warm-up of each.  Run plain first, then under ncu (see B200_PROFILING.md)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "xoshiro256starstar"
spec = P.get_spec(name)
n, T = (1 << 20), 1024
out = torch.empty((n, T), dtype=torch.uint64 if spec.kind.w == 64 else torch.uint32, device="cuda")
for _ in range(2):
    sub = D.Substreams.from_seed(spec, 42, n)
    sub.fill(T, out=out)
    sub.checksum(T)
torch.cuda.synchronize()
print("ok")

"""Short workload for ncu launch lists of substream initialisation (K1 + K1t):
warm-up call, then one timed-shape call of Substreams.from_seed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "xoshiro256starstar"
spec = P.get_spec(name)
n = (1 << 20) if spec.kind.w == 64 else (1 << 21)
for _ in range(2):
    D.Substreams.from_seed(spec, 42, n)
torch.cuda.synchronize()
print("ok")

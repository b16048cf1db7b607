"""Short workload for the ncu pipe counts of kernel K4 (fused consumer) on
config 2 (xoshiro256**, 2^20 substreams x 1024): sum+xor, exact, exact+f64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec(sys.argv[1] if len(sys.argv) > 1 else "xoshiro256starstar")
sub = D.Substreams.from_seed(spec, 42, 1 << 20)
raw = torch.empty(48, dtype=torch.uint8, device="cuda")
for kw in (dict(exact=False), dict(exact=True), dict(exact=True, f64=True)):
    sub.checksum_async(1024, result=raw, **kw)
torch.cuda.synchronize()
print("ok")

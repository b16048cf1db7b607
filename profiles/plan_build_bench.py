"""Host cost of a new init plan (first fill of a single stream with a fresh
length T: characteristic polynomial cached, x^J and the direct polynomials
new) against the warm call, per SLP_PLAN_DIRECT.  Wall-clock ms."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

for name in ["xoroshiro1024starstar", "xoshiro512starstar", "xoshiro256starstar"]:
    spec = P.get_spec(name)
    one = D.Substreams.from_seed(spec, 42, 1)
    out = torch.empty((1, 1 << 26), dtype=torch.uint64, device="cuda")
    one.fill(1 << 26, out=out)  # char poly, kernels, allocator warm
    torch.cuda.synchronize()
    first, warm = [], []
    for i in range(1, 6):
        T = (1 << 26) - 4096 * i  # fresh stride every time
        o = out[:, :T]
        for lst in (first, warm):
            t0 = time.perf_counter()
            one.fill(T, out=o)
            torch.cuda.synchronize()
            lst.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"direct": os.environ.get("SLP_PLAN_DIRECT", "default"), "name": name,
                      "first_ms": round(min(first), 3), "first_ms_max": round(max(first), 3),
                      "warm_ms": round(min(warm), 3)}), flush=True)

"""Fused checksum (K4) rate over the substream count at T = 8192, for split
thresholds SLP_FUSED_SPLIT_NMAX in argv (read on every call).  One JSON line
per (threshold, n)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec(os.environ.get("K4_GEN", "xoshiro256starstar"))
T = 8192
for nmax in [int(a) for a in sys.argv[1:]] or [1 << 15]:
    os.environ["SLP_FUSED_SPLIT_NMAX"] = str(nmax)
    for n in [1 << 12, 1 << 14, 1 << 15, 1 << 16, 1 << 17, 1 << 18, 1 << 20]:
        sub = D.Substreams.from_seed(spec, 42, n)
        sub.checksum_async(T)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sub.checksum_async(T)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"nmax": nmax, "n": n, "T": T, "ms": ms, "outputs_per_s": n * T / ms * 1e3}), flush=True)

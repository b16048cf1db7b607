"""HWD consumer (K6) rate per generator for A/B builds (SLP_LIB=variants/...):
1e12 bytes of generator output, k = 8, w = 64.  One JSON line per generator."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_01407_b200 import hwd  # noqa: E402

GENS = sys.argv[1:] or ["xoshiro256starstar", "xoshiro256plusplus", "xoroshiro128plusplus", "xoroshiro128starstar",
                        "xoshiro512starstar", "xoroshiro1024plusplus", "xoroshiro128plus"]
hwd.run_generator("xoshiro256plus", hwd.HwdConfig(w=64, k=8, byte_limit=8 * 10 ** 6), seed=1)  # warm-up
for name in GENS:
    cfg = hwd.HwdConfig(w=64, k=8, byte_limit=10 ** 12)
    best = None
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = hwd.run_generator(name, cfg, seed=1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    print(json.dumps({"lib": os.path.basename(os.environ.get("SLP_LIB") or "main"), "generator": name,
                      "status": rep.status, "signature": rep.faulty_signature, "p_value": rep.p_value,
                      "seconds": round(best, 4), "values_per_s": rep.values / best}), flush=True)

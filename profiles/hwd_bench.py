"""GPU HWD consumer timings on the paper rows (test values/s, bytes/s)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_01407_b200 import hwd  # noqa: E402

ROWS = [
    ("xorshift128plus", dict(w=64, k=8, byte_limit=int(2.4e10), mode="transitional")),
    ("xoshiro256starstar", dict(w=64, k=8, byte_limit=int(1e10))),
    ("xoshiro256starstar", dict(w=64, k=8, byte_limit=int(1e12))),
    ("xoroshiro128plus", dict(w=64, k=8, byte_limit=int(1e12))),
    ("xoshiro128plusplus", dict(w=32, k=8, byte_limit=int(4e11))),
]
hwd.run_generator("xoshiro256plus", hwd.HwdConfig(w=64, k=8, byte_limit=8 * 10 ** 6), seed=1)  # warm-up
for name, kw in ROWS:
    cfg = hwd.HwdConfig(**kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = hwd.run_generator(name, cfg, seed=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"generator": name, "config": kw, "status": rep.status, "bytes": rep.bytes_processed,
                      "p_value": rep.p_value, "signature": rep.faulty_signature, "seconds": round(dt, 3),
                      "GB_per_s": round(rep.bytes_processed / dt / 1e9, 1),
                      "values_per_s": rep.values / dt, "checkpoints": len(rep.history)}), flush=True)

"""GPU HWD counting rate over k (xoshiro256**, standard mode): shared-memory
cells (k <= 9), sliced cells (k = 10, 11) and global 64-bit atomics
(k >= 12); the counting kernel alone (hwd._GpuCounter.count, one range),
not the checkpoint evaluation.  One JSON line per k.  (A packed
one-atomic-per-value variant, SLP_HWD_PACK, measured 15-30% slower at
k = 12-14 and was dropped; its "pack" column in round1_hwd_k_bench.jsonl
is that experiment.)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_01407_b200 import hwd  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402

spec = P.get_spec("xoshiro256starstar")
for k, n in [(8, 4 * 10 ** 10), (10, 10 ** 10), (11, 4 * 10 ** 9), (12, 10 ** 9), (13, 4 * 10 ** 8),
             (14, 2 * 10 ** 8)]:
    for pack in ["-"]:
        cfg = hwd.HwdConfig(w=64, k=k)
        ctr = hwd._GpuCounter(spec, 1, cfg)
        ctr.count(0, 10 ** 6)  # warm-up (plans, tables)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctr.count(10 ** 6, 10 ** 6 + n)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"k": k, "pack": pack, "values": n, "seconds": round(dt, 4), "values_per_s": n / dt}),
              flush=True)

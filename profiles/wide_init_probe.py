"""Round 2: wide-engine initialisation (xoroshiro1024, xoshiro512): init of
2^20 and 2^15 substreams, and the one-long-stream fill whose segment split
runs the same plan machinery (2 GiB).  Warm (plans and tables built), CUDA
events, best of 3 x 5.  Knobs: SLP_PLAN_DIRECT, SLP_INIT_TABLES."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


tag = {k: os.environ.get(k) for k in ("SLP_PLAN_DIRECT", "SLP_INIT_TABLES")}
for name in ("xoroshiro1024starstar", "xoshiro512starstar", "xoshiro256starstar"):
    spec = P.get_spec(name)
    r = {"name": name, **tag}
    for n in (1 << 20, 1 << 15):
        r[f"init_{n}_ms"] = round(timeit(lambda: D.Substreams.from_seed(spec, 42, n)), 4)
    one = D.Substreams.from_seed(spec, 42, 1)
    out = torch.empty((1, 1 << 28), dtype=torch.uint64, device="cuda")
    ms = timeit(lambda: one.fill(1 << 28, out=out), 3)
    r["one_stream_2GiB_ms"] = round(ms, 4)
    r["one_stream_TB_s"] = round((1 << 31) / ms / 1e9, 3)
    print(json.dumps(r), flush=True)
    del out

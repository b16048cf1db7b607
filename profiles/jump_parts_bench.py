"""K1 lane-split A/B (SLP_JUMP_PARTS=1 off, unset = auto): single-stream fills
of the wide engines (segment split: K1 jumps dominate the set-up), default
LanedStream geometry, and small substream inits.  One JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402


def timeit(fn, reps=5):
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


mode = os.environ.get("SLP_JUMP_PARTS", "auto") + ("/direct=" + os.environ["SLP_PLAN_DIRECT"] if os.environ.get("SLP_PLAN_DIRECT") else "")
for name in (sys.argv[1:] or ["xoroshiro1024starstar", "xoroshiro1024plusplus", "xoshiro512starstar", "xoshiro256starstar"]):
    spec = P.get_spec(name)
    for T in (1 << 28, 1 << 24):
        one = D.Substreams.from_seed(spec, 42, 1)
        out = torch.empty((1, T), dtype=torch.uint64, device="cuda")
        ms = timeit(lambda: one.fill(T, out=out))
        print(json.dumps({"parts": mode, "case": "one stream fill", "name": name, "T": T, "ms": round(ms, 4),
                          "TBps": round(T * 8 / ms / 1e9, 3)}), flush=True)
        del out
    ms = timeit(lambda: D.Substreams.from_seed(spec, 42, 1).checksum(1 << 28))
    print(json.dumps({"parts": mode, "case": "one stream checksum 2^28", "name": name, "ms": round(ms, 4)}), flush=True)
    for n in (4096, 1 << 15, 1 << 17, 1 << 20):
        ms = timeit(lambda: D.Substreams.from_seed(spec, 42, n))
        print(json.dumps({"parts": mode, "case": "init", "name": name, "n": n, "ms": round(ms, 4)}), flush=True)

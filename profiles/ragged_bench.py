"""Ragged rows (T not a multiple of the fill tile): stream-major store rate
for T around the tile sizes, ~8 GB of output per call, warm, CUDA events
(best of 3 batches).  One JSON line per (generator, kind, T)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

TS = [int(t) for t in os.environ.get("RAGGED_TS", "64,100,127,1000,1024,1055,1100,1151,1500,2047,4000").split(",")]
NAMES = sys.argv[1:] or ["xoshiro256starstar", "xoroshiro128plus", "xoroshiro1024plusplus", "xoshiro128starstar"]


def timeit(fn, reps=10):
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


for name in NAMES:
    spec = P.get_spec(name)
    kinds = ["native", "f64"] if spec.kind.w == 64 else ["native", "f32"]
    for kind in kinds:
        es = 8 if spec.kind.w == 64 else 4
        for T in TS:
            n = max(1 << 18, (8 << 30) // (T * es) // 32 * 32)
            sub = D.Substreams.from_seed(spec, 42, n)
            out = torch.empty((n, T), dtype=D._out_dtype(spec, kind), device="cuda")
            ms = timeit(lambda: D.fill(spec, sub.states, T, out=out, kind=kind))
            print(json.dumps({"name": name, "kind": kind, "n": n, "T": T, "ms": ms,
                              "TB_s": n * T * es / ms / 1e9}), flush=True)
            del out, sub

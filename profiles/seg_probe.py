"""Round 2 probe: does the stream-major write pattern, not generation, cap
k_fill?  Same 8 GiB of xoshiro256** outputs written as (n, T) stream-major
rows for T = 64 .. 1024: with T = 128 a warp's 32 rows are one contiguous
32 KiB block (the pattern a segment-parallel config-2 fill would write),
with T = 1024 a warp has 32 rows 8 KiB apart in flight.  Warm, CUDA events,
best of 3 x 10 launches.  One JSON line each (TB/s of output bytes and of
output + state bytes)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402


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


names = sys.argv[1:] or ["xoshiro256starstar"]
TOTAL = 1 << 30
for name in names:
    spec = P.get_spec(name)
    kb = spec.kind.k * spec.kind.w // 8
    es = spec.kind.w // 8
    for T in (64, 128, 256, 512, 1024):
        n = TOTAL // T
        sub = D.Substreams.from_seed(spec, 42, n)
        out = torch.empty((n, T), dtype=torch.uint64 if es == 8 else torch.uint32, device="cuda")
        ms = timeit(lambda: D.fill(spec, sub.states, T, out=out))
        ob = n * T * es
        print(json.dumps({"name": name, "n": n, "T": T, "ms": round(ms, 4), "out_TB_s": round(ob / ms / 1e9, 3),
                          "total_TB_s": round((ob + 2 * n * kb) / ms / 1e9, 3)}), flush=True)
        del out, sub
        torch.cuda.empty_cache()
    # write-only reference on the same tensor size
    x = torch.empty(TOTAL, dtype=torch.int64 if es == 8 else torch.int32, device="cuda")
    ms = timeit(lambda: x.fill_(1))
    print(json.dumps({"name": "fill_", "bytes": TOTAL * es, "TB_s": round(TOTAL * es / ms / 1e9, 3)}), flush=True)
    del x

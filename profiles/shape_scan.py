"""Stream-major fill rate over (substreams, row length) for xoshiro256**:
where the one-thread-per-substream fill runs out of parallelism and where the
segment split takes over.  Warm, CUDA events, best of 3.  One JSON line each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

NAME = sys.argv[1] if len(sys.argv) > 1 else "xoshiro256starstar"
NS = [1 << 10, 1 << 12, 1 << 14, 1 << 15, 1 << 16, 1 << 17, 1 << 18]
TS = [512, 1024, 2048, 4096, 16384]


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


spec = P.get_spec(NAME)
for n in NS:
    sub = D.Substreams.from_seed(spec, 42, n)
    for T in TS:
        if n * T * 8 > (8 << 30):
            continue
        out = torch.empty((n, T), dtype=torch.uint64, device="cuda")
        ms = timeit(lambda: D.fill(spec, sub.states, T, out=out))
        print(json.dumps({"name": NAME, "n": n, "T": T, "J": D._split_factor(spec, n, T, "stream", T), "ms": ms,
                          "TB_s": n * T * 8 / ms / 1e9}), flush=True)
        del out

"""Round 2: the shapes VERDICT r1 item 6 lists as slow, measured on the
current build.  Output bytes / kernel time (CUDA events, warm, best of 3 x
5 launches).  One JSON line per case."""
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


def case(label, name, n, T, layout="stream", ld_pad=0, kind="native"):
    spec = P.get_spec(name)
    sub = D.Substreams.from_seed(spec, 42, n)
    es = 8 if (spec.kind.w == 64 or kind in ("u64", "f64")) else 4
    dt = {8: torch.uint64, 4: torch.uint32}[es] if kind in ("native", "u64") else \
        {"f64": torch.float64, "f32": torch.float32}[kind]
    rows, cols = (n, T) if layout == "stream" else (T, n)
    buf = torch.empty((rows, cols + ld_pad), dtype=dt, device="cuda")
    out = buf[:, :cols]
    ms = timeit(lambda: D.fill(spec, sub.states, T, out=out, layout=layout, kind=kind))
    print(json.dumps({"case": label, "name": name, "n": n, "T": T, "layout": layout, "ld_pad": ld_pad, "kind": kind,
                      "ms": round(ms, 4), "TB_s": round(n * T * es / ms / 1e9, 3)}), flush=True)


N = 1 << 20
case("pm aligned (TMA)", "xoshiro256starstar", N, 1024, "position")
case("pm odd n (FILL_POS)", "xoshiro256starstar", N + 1, 1024, "position")
case("pm odd n (FILL_POS)", "xoroshiro128plus", N + 1, 1024, "position")
case("pm odd n u32 (FILL_POS)", "xoshiro128starstar", 2 * N + 1, 1024, "position")
case("pm padded pitch +1", "xoshiro256starstar", N, 1024, "position", ld_pad=1)
case("sm odd T (TMA_G)", "xoshiro256starstar", N, 1023)
case("sm odd T u32 (TMA_G)", "xoshiro128starstar", 2 * N, 1023)
case("sm few long, contiguous (split)", "xoshiro256starstar", 16, 1 << 24)
case("sm few long, padded pitch (no split)", "xoshiro256starstar", 16, 1 << 24, ld_pad=16)
case("pm few long (no split)", "xoshiro256starstar", 16, 1 << 22, "position")
case("sm one long (split)", "xoroshiro1024starstar", 1, 1 << 28)
case("sm one long (split)", "xoshiro256starstar", 1, 1 << 28)
spec = P.get_spec("xoroshiro1024starstar")
D.Substreams.from_seed(spec, 42, N)
ms = timeit(lambda: D.Substreams.from_seed(spec, 42, N), 3)
print(json.dumps({"case": "xoroshiro1024 init 2^20 substreams (K1 + K1t)", "ms": round(ms, 4)}), flush=True)

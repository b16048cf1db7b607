"""Store pacing sweep (round 2): k_fill at BASELINE config-2 shapes with the
aggregate store-pacing target (slp_set_fill_pace, GB/s) swept; 0 = unpaced.
Each target is timed between two unpaced runs on the same box (CUDA events,
`--launches` back-to-back 8 GiB launches after 3 warm-ups).  One JSON line per
(case, target); also the live write-only ceiling (torch fill_ of the buffer).

  python profiles/pace_sweep.py [--launches 30] [--targets 6000,6100,...] [--cases c2,c2f64,...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import _native  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

CASES = {
    # name: (generator, substreams, T, kind, layout)
    "c2": ("xoshiro256starstar", 1 << 20, 1024, "native", "stream"),
    "c2f64": ("xoshiro256starstar", 1 << 20, 1024, "f64", "stream"),
    "c3": ("xoroshiro128plus", 1 << 20, 1024, "f64", "stream"),
    "c4": ("xoshiro128starstar", 1 << 21, 1024, "f32", "stream"),
    "c4u": ("xoroshiro64star", 1 << 21, 1024, "native", "stream"),
    "x512": ("xoshiro512starstar", 1 << 20, 1024, "native", "stream"),
    "x1024": ("xoroshiro1024plusplus", 1 << 20, 1024, "native", "stream"),
    "pm": ("xoshiro256starstar", 1 << 20, 1024, "native", "position"),
    "t64": ("xoshiro256starstar", 1 << 24, 64, "native", "stream"),
    "t128": ("xoshiro256starstar", 1 << 23, 128, "native", "stream"),
    "t256": ("xoshiro256starstar", 1 << 22, 256, "native", "stream"),
    "t2048": ("xoshiro256starstar", 1 << 19, 2048, "native", "stream"),
    "oddT": ("xoshiro256starstar", 1 << 20, 1023, "native", "stream"),
    "oddT32": ("xoshiro128starstar", 1 << 21, 1023, "native", "stream"),
    "pmf64": ("xoroshiro128plus", 1 << 20, 1024, "f64", "position"),
    "pm1024": ("xoroshiro1024plusplus", 1 << 20, 1024, "native", "position"),
    "x1024na": ("xoroshiro1024plusplus", 1 << 20, 1024, "native", "stream", 0, False),
    "x512na": ("xoshiro512starstar", 1 << 20, 1024, "native", "stream", 0, False),
    "pm32": ("xoshiro128starstar", 1 << 21, 1024, "native", "position"),
    "pmf32": ("xoshiro128starstar", 1 << 21, 1024, "f32", "position"),
    # odd pitch (one element of padding per row): CTA-staged position-major path
    "pmodd": ("xoshiro256starstar", 1 << 20, 1024, "native", "position", 1),
    "pmodd32": ("xoshiro128starstar", 1 << 21, 1024, "native", "position", 1),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=30)
    ap.add_argument("--targets", default="6000,6200,6400,6500,6600,6700,6800,6900,7000,7200")
    ap.add_argument("--cases", default="c2")
    a = ap.parse_args()
    lib = _native.lib()
    targets = [int(x) for x in a.targets.split(",")]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for case in a.cases.split(","):
        gen, n, T, kind, layout = CASES[case][:5]
        pad = CASES[case][5] if len(CASES[case]) > 5 else 0
        adv = CASES[case][6] if len(CASES[case]) > 6 else True  # False: no state write-back
        spec = P.get_spec(gen)
        sub = D.Substreams.from_seed(spec, 42, n)
        out = sub.fill(T, kind=kind, layout=layout)
        if pad:
            rows, cols = out.shape
            out = torch.empty((rows, cols + pad), dtype=out.dtype, device=out.device)[:, :cols]
        nbytes = out.numel() * out.element_size()

        def timed(target):
            lib.slp_set_fill_pace(target)
            for _ in range(3):
                sub.fill(T, kind=kind, layout=layout, out=out, advance=adv)
            ev0.record()
            for _ in range(a.launches):
                sub.fill(T, kind=kind, layout=layout, out=out, advance=adv)
            ev1.record()
            torch.cuda.synchronize()
            return ev0.elapsed_time(ev1) / a.launches

        for _ in range(2):
            out.fill_(1)
        ev0.record()
        for _ in range(10):
            out.fill_(1)
        ev1.record()
        torch.cuda.synchronize()
        wo = nbytes / (ev0.elapsed_time(ev1) / 10 / 1e3) / 1e9
        for t in targets:
            base0 = timed(0)
            ms = timed(t)
            base1 = timed(0)
            base = (base0 + base1) / 2
            print(json.dumps({"case": case, "generator": gen, "n": n, "T": T, "kind": kind, "layout": layout,
                              "target_gbps": t, "ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1),
                              "unpaced_ms": round(base, 4), "unpaced_GBps": round(nbytes / base / 1e6, 1),
                              "speedup": round(base / ms, 4), "write_only_gbps": round(wo, 1)}), flush=True)
        lib.slp_set_fill_pace(0)
        del out, sub
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

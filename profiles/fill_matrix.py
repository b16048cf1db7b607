"""Fill-kernel throughput matrix for the tile-configuration tuning
(profiles/tune_fill.py): for every generator, the three k_fill kinds --
store native, store converted (f64 for w=64, f32 for w=32), store +
checksum in one pass (converted) -- at config-2 sizes (2^20 substreams x
1024 for w=64, 2^21 x 1024 for w=32), CUDA events, warm.  The library is
whatever SLP_LIB points at.  One JSON line per (generator, kind)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(3):  # best of 3 batches: robust to one slow batch
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*")
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--tag", default=os.environ.get("SLP_LIB", "default"))
    a = ap.parse_args()
    names = a.names or P.registry_names(True)
    T = 1024
    for name in names:
        spec = P.get_spec(name)
        w = spec.kind.w
        n = (1 << 20) if w == 64 else (1 << 21)
        sub = D.Substreams.from_seed(spec, 42, n)
        outs = n * T
        fkind = "f64" if w == 64 else "f32"
        o = torch.empty((n, T), dtype=torch.uint64 if w == 64 else torch.uint32, device="cuda")
        f = torch.empty((n, T), dtype=torch.float64 if w == 64 else torch.float32, device="cuda")
        cases = [("native", lambda: sub.fill(T, out=o)),
                 ("convert", lambda: sub.fill(T, out=f, kind=fkind)),
                 ("checksum", lambda: D.fill_checksum(spec, sub.states, T, out=f, kind=fkind))]
        for kind, fn in cases:
            ms = timeit(fn, a.reps)
            print(json.dumps({"tag": a.tag, "name": name, "kind": kind, "out_per_s": outs / ms * 1e3}), flush=True)
        del o, f, sub
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

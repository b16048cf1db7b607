"""Quick per-kernel timings (CUDA events, warm, 8 GiB outputs >> L2) for one or
more generators: store fill (u64/u32 native, f64/f32), fused checksum
(int / exact / f64) and substream init.  Prints one JSON line per generator.
usage: python profiles/microbench.py [name ...] [--n N] [--T T] [--reps R]"""
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
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["xoshiro256starstar"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--T", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--skip-store", action="store_true")
    a = ap.parse_args()
    for name in a.names:
        spec = P.get_spec(name)
        w = spec.kind.w
        n = a.n or ((1 << 20) if w == 64 else (1 << 21))
        T = a.T
        outs = n * T
        res = {"name": name, "n": n, "T": T}
        res["init_ms"] = timeit(lambda: D.Substreams.from_seed(spec, 42, n), 5)
        sub = D.Substreams.from_seed(spec, 42, n)
        if not a.skip_store:
            out = torch.empty((n, T), dtype=torch.uint64 if w == 64 else torch.uint32, device="cuda")
            ms = timeit(lambda: sub.fill(T, out=out), a.reps)
            res["store_ms"] = ms
            res["store_out_per_s"] = outs / ms * 1e3
            res["store_GBps"] = outs * (w // 8) / ms / 1e6
            del out
            fo = torch.empty((n, T), dtype=torch.float64 if w == 64 else torch.float32, device="cuda")
            ms = timeit(lambda: sub.fill(T, out=fo, kind="f64" if w == 64 else "f32"), a.reps)
            res["store_float_out_per_s"] = outs / ms * 1e3
            del fo
        raw = torch.empty(48, dtype=torch.uint8, device="cuda")
        for label, kw in [("fused_int", dict(exact=False)), ("fused_exact", dict(exact=True)),
                          ("fused_f64", dict(exact=True, f64=True))]:
            ms = timeit(lambda: sub.checksum_async(T, result=raw, **kw), a.reps)
            res[label + "_out_per_s"] = outs / ms * 1e3
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

"""A/B of K4 (k_fused) builds that move shift / multiply / rotation sites to the
FMA pipe (Makefile variants with -DSLP_FUSED_MASK[2]=...): per library, per
generator, the three fused modes at config-2 size plus a checksum of a small
case, which must be identical in every build.  One process per library.
usage: python profiles/ab_fused_mask.py [--rounds R] lib.so [lib.so ...]"""
import json
import os
import subprocess
import sys

GENS = ["xoshiro256starstar", "xoshiro256plusplus", "xoshiro256plus", "xoroshiro128plus", "xoroshiro128plusplus",
        "xoroshiro128starstar", "xoshiro512starstar", "xoshiro512plusplus", "xoroshiro1024plusplus",
        "xoroshiro1024starstar", "xoroshiro1024star"]


def one():
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    import paper_1805_01407_b200 as P
    from paper_1805_01407_b200 import device as D

    def timeit(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for name in GENS:
        spec = P.get_spec(name)
        small = D.Substreams.from_seed(spec, 42, 4099)
        c = small.checksum(1037, f64=True)
        c2 = D.Substreams.from_seed(spec, 42, 4099).checksum(1037, exact=False)
        n, T = 1 << 20, 1024
        sub = D.Substreams.from_seed(spec, 42, n)
        raw = torch.empty(48, dtype=torch.uint8, device="cuda")
        res = {"lib": os.path.basename(os.environ.get("SLP_LIB", "main")), "name": name,
               "check": "%x/%x/%x/%x" % (c.sum, c.xor, c.mant, c2.xor)}
        for label, kw in [("int", dict(exact=False)), ("exact", dict(exact=True)), ("f64", dict(exact=True, f64=True))]:
            ms = timeit(lambda: sub.checksum_async(T, result=raw, **kw))
            res[label] = round(n * T / ms * 1e3 / 1e9, 1)  # G outputs/s
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        one()
    else:
        args = sys.argv[1:]
        rounds = 2
        if args[0] == "--rounds":
            rounds = int(args[1])
            args = args[2:]
        for _ in range(rounds):
            for lib in args:
                env = dict(os.environ)
                if lib != "main":
                    env["SLP_LIB"] = os.path.abspath(lib)
                subprocess.run([sys.executable, os.path.abspath(__file__), "--one"], env=env, check=False)

"""BASELINE configs 3 and 4 at full size on one GPU (CUDA events, warm):
store (native / float), store + fused checksum in one pass, fused checksum
only.  Prints one JSON line per generator."""
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
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


CASES = [("c3", n, 42, 1 << 21, "f64") for n in ("xoroshiro128plus", "xoroshiro128plusplus", "xoroshiro128starstar")]
CASES += [("c4", n, 7, 1 << 22, "f32") for n in ("xoshiro128starstar", "xoshiro128plusplus", "xoroshiro64star",
                                                  "xoroshiro64starstar")]
T = 1024
for cfg, name, seed, n, fkind in CASES:
    spec = P.get_spec(name)
    sub = D.Substreams.from_seed(spec, seed, n)
    outs = n * T
    wdt = torch.uint64 if spec.kind.w == 64 else torch.uint32
    fdt = torch.float64 if fkind == "f64" else torch.float32
    res = {"config": cfg, "generator": name, "substreams": n, "T": T}
    o = torch.empty((n, T), dtype=wdt, device="cuda")
    res["store_native_out_per_s"] = outs / timeit(lambda: sub.fill(T, out=o)) * 1e3
    del o
    f = torch.empty((n, T), dtype=fdt, device="cuda")
    ms = timeit(lambda: sub.fill(T, out=f, kind=fkind))
    res[f"store_{fkind}_out_per_s"] = outs / ms * 1e3
    res[f"store_{fkind}_GBps"] = outs * f.element_size() / ms / 1e6
    ms = timeit(lambda: D.fill_checksum(spec, sub.states, T, out=f, kind=fkind))
    res[f"store_{fkind}_plus_checksum_out_per_s"] = outs / ms * 1e3
    del f
    raw = torch.empty(48, dtype=torch.uint8, device="cuda")
    res["fused_exact_f64_out_per_s"] = outs / timeit(lambda: sub.checksum_async(T, f64=True, result=raw)) * 1e3
    res["fused_int_out_per_s"] = outs / timeit(lambda: sub.checksum_async(T, exact=False, result=raw)) * 1e3
    print(json.dumps(res), flush=True)

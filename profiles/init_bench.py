"""Substream initialisation (kernels K1 / K1t) timing: Substreams.from_seed for
2^20 (w=64) or 2^21 (w=32) substreams, warm (plan, device polynomials and
jump tables built by a first call), CUDA events, with the table-driven radix
rounds (K1t) on and off (SLP_INIT_TABLES).  One JSON line per generator."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

NAMES = sys.argv[1:] or ["xoroshiro128plus", "xoshiro256starstar", "xoshiro512starstar", "xoroshiro1024starstar",
                         "xoroshiro64star", "xoshiro128starstar"]


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for name in NAMES:
    spec = P.get_spec(name)
    n = (1 << 20) if spec.kind.w == 64 else (1 << 21)
    res = {"name": name, "substreams": n}
    for tag, flag in (("tables", "1"), ("poly", "0")):
        os.environ["SLP_INIT_TABLES"] = flag
        res[f"init_ms_{tag}"] = timeit(lambda: D.Substreams.from_seed(spec, 42, n))
    # config-5 shape: 8 long-jump blocks x 2^18 substreams
    os.environ["SLP_INIT_TABLES"] = "1"
    res["init_ms_8x2^18_tables"] = timeit(lambda: D.Substreams.from_seed(spec, 42, 1 << 18, blocks=8))
    os.environ["SLP_INIT_TABLES"] = "0"
    res["init_ms_8x2^18_poly"] = timeit(lambda: D.Substreams.from_seed(spec, 42, 1 << 18, blocks=8))
    print(json.dumps(res), flush=True)

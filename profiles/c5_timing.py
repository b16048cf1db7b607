"""Config-5 job breakdown: host block jumps + K1 init + K4 fused checksum."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0):9.2f} ms", flush=True)
    return r


for name in ("xoshiro512starstar", "xoroshiro1024plusplus"):
    spec = P.get_spec(name)
    g = P.Generator.from_seed(spec, 42)
    S, T = 1 << 18, 1 << 13
    t(f"{name} first init (plan build)", lambda: D.Substreams.from_generator(g, S, blocks=8))
    sub = t(f"{name} init 8 x 2^18", lambda: D.Substreams.from_generator(g, S, blocks=8))
    t(f"{name} fused exact 2^34", lambda: sub.checksum(T))
    sub = D.Substreams.from_generator(g, S, blocks=8)
    t(f"{name} fused int 2^34", lambda: sub.checksum(T, exact=False))
    t(f"{name} per-block init", lambda: [D.Substreams.from_generator(g, S, first_block=b) for b in range(8)])

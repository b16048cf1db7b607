"""Store + checksum in one pass (K2 CSUM kind) per generator, for A/B builds
(SLP_LIB=variants/...): outputs/s at config-2 size.
usage: [SLP_LIB=lib.so] python profiles/ab_fill_csum.py [name ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

names = sys.argv[1:] or ["xoshiro256starstar", "xoroshiro128starstar", "xoshiro512starstar", "xoroshiro1024starstar",
                         "xoroshiro1024star", "xoroshiro128star"]
for name in names:
    spec = P.get_spec(name)
    n, T = 1 << 20, 1024
    sub = D.Substreams.from_seed(spec, 42, n)
    out = torch.empty((n, T), dtype=torch.uint64, device="cuda")
    D.fill_checksum(spec, sub.states, T, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _, c = D.fill_checksum(spec, sub.states, T, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"lib": os.path.basename(os.environ.get("SLP_LIB") or "main"), "name": name,
                      "store_checksum_out_per_s": n * T / ms * 1e3, "xor": hex(c.xor)}), flush=True)

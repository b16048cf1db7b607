"""Fused checksum (K4) of few long substreams, with and without the segment split
(SLP_SPLIT=0 disables it; read on every call).  One JSON line per case."""
import sys, json, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
for name in ["xoshiro256starstar", "xoroshiro1024plusplus"]:
    spec = P.get_spec(name)
    for n, T in [(1, 1 << 28), (16, 1 << 24), (1000, 1 << 18)]:
        for split in (True, False):
            os.environ["SLP_SPLIT"] = "1" if split else "0"
            sub = D.Substreams.from_seed(spec, 42, n)
            sub.checksum(T)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); c = sub.checksum_async(T); e1.record(); e1.synchronize()
            ms = e0.elapsed_time(e1)
            print(json.dumps({"name": name, "n": n, "T": T, "split": split, "ms": ms, "outputs_per_s": n * T / ms * 1e3}), flush=True)

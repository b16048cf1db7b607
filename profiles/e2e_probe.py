"""Round 2: where the e2e leg (seed -> 8 GiB of outputs in pinned host memory)
loses against the raw 56 GB/s PCIe D2H: fill_to_host with 2/3/4 device
buffers and 64 MiB .. 1 GiB slices, against one fill + one 8 GiB copy."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

spec = P.get_spec("xoshiro256starstar")
N, T = 1 << 20, 1024
host = torch.empty((N, T), dtype=torch.uint64, pin_memory=True)
sub = D.Substreams.from_seed(spec, 42, N)


def run(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return N * T * 8 / best / 1e9


for nb in (2, 3, 4):
    for sl in (1 << 13, 1 << 15, 1 << 17):
        bufs = [torch.empty((sl, T), dtype=torch.uint64, device="cuda") for _ in range(nb)]
        gbs = run(lambda: D.fill_to_host(spec, sub.states, T, host, slice_streams=sl, _bufs=bufs))
        print(json.dumps({"bufs": nb, "slice_MiB": sl * T * 8 >> 20, "GBps": round(gbs, 2)}), flush=True)
        del bufs
full = torch.empty((N, T), dtype=torch.uint64, device="cuda")


def whole():
    sub.fill(T, out=full)
    host.copy_(full, non_blocking=True)


print(json.dumps({"fill_then_one_copy": True, "GBps": round(run(whole), 2)}), flush=True)

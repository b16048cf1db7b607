import sys, time, json
sys.path.insert(0, "/root/repo")
import torch
import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
spec = P.get_spec("xoshiro256starstar")
N, T = 1 << 20, 1024
out = torch.empty((N, T), dtype=torch.uint64, device="cuda")
sub = D.Substreams.from_seed(spec, 42, N)
for _ in range(30): sub.fill(T, out=out)
torch.cuda.synchronize()
host = torch.empty((N, T), dtype=torch.uint64, pin_memory=True)
bufs = [torch.empty((1 << 15, T), dtype=torch.uint64, device="cuda") for _ in range(2)]
del out
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s2 = D.Substreams.from_seed(spec, 42, N)
    D.fill_to_host(spec, s2.states, T, host, _bufs=bufs)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"step": i, "ms": round(dt * 1e3, 1), "GBps": round(N * T * 8 / dt / 1e9, 1)}), flush=True)

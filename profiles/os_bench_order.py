import sys, time, json
sys.path.insert(0, "/root/repo")
import torch
import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
spec = P.get_spec("xoshiro256starstar")
N, T = 1 << 20, 1024
def os_run(tag):
    t0 = time.perf_counter(); ts = []; last = t0
    for c in P.output_stream(spec, 43, 1 << 28, lanes=1 << 16, lane_len=1024):
        del c
        now = time.perf_counter(); ts.append(round((now - last) * 1e3, 1)); last = now
    print("warm", ts)
    t0 = time.perf_counter(); got = 0; pooled = 0; ts = []; last = t0
    for c in P.output_stream(spec, 42, 1 << 30, lanes=1 << 16, lane_len=1024):
        got += c.size; pooled += isinstance(c.base, torch.Tensor)
        now = time.perf_counter(); ts.append(round((now - last) * 1e3, 1)); last = now
    dt = time.perf_counter() - t0
    print(tag, got / dt / 1e9, pooled, ts, flush=True)
os_run("fresh")
host = torch.empty((N, T), dtype=torch.uint64, pin_memory=True)
bufs = [torch.empty((1 << 15, T), dtype=torch.uint64, device="cuda") for _ in range(2)]
s2 = D.Substreams.from_seed(spec, 42, N)
D.fill_to_host(spec, s2.states, T, host, _bufs=bufs); torch.cuda.synchronize()
del host, bufs
os_run("after e2e")
outd = torch.empty((N, T), dtype=torch.uint64, device="cuda")
res_host = torch.empty(1, dtype=torch.uint64, pin_memory=True)
s3 = D.Substreams.from_seed(spec, 42, N); s3.fill(T, out=outd); res_host.copy_(outd[-1, -1:], non_blocking=True)
torch.cuda.synchronize(); del outd
os_run("after dev")

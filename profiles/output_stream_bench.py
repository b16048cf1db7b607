import time, sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1805_01407_b200 as P
spec = P.get_spec("xoshiro256starstar")
total = 1 << 30
for lanes, lane_len in [(4096, 4096), (16384, 4096), (65536, 1024)]:
    it = P.output_stream(spec, 42, total, lanes=lanes, lane_len=lane_len)
    first = next(it)  # warm (plans)
    t = time.perf_counter(); n = first.size
    for c in it:
        n += c.size
    dt = time.perf_counter() - t
    print("output_stream", lanes, lane_len, "values/s %.3g" % ((n - first.size) / dt), "GB/s %.1f" % ((n - first.size) * 8 / dt / 1e9))
# raw host paths for a 128 MB chunk
x = torch.empty(1 << 24, dtype=torch.uint64, device="cuda")
for name, fn in [("cpu().numpy()", lambda: x.cpu().numpy()),
                 ("pinned copy", None)]:
    if fn is None:
        h = torch.empty(1 << 24, dtype=torch.uint64, pin_memory=True)
        fn = lambda: h.copy_(x)
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
    print(name, "GB/s %.1f" % (x.numel() * 8 / dt / 1e9))
h = torch.empty(1 << 24, dtype=torch.uint64, pin_memory=True)
t = time.perf_counter()
for _ in range(10):
    a = np.empty(1 << 24, dtype=np.uint64); a[:] = h.numpy()
dt = (time.perf_counter() - t) / 10
print("pinned -> fresh numpy memcpy GB/s %.1f" % ((1 << 27) / dt / 1e9))
t = time.perf_counter()
for _ in range(10):
    a = np.empty(1 << 24, dtype=np.uint64); torch.from_numpy(a).copy_(x)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
print("D2H into fresh numpy (pageable) GB/s %.1f" % ((1 << 27) / dt / 1e9))
import os; print("cpus", os.cpu_count())

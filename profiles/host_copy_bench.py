"""Host-side delivery of a 128 MB chunk as a FRESH numpy array (the
LanedStream.chunks contract): single-threaded vs threaded copies out of a
pinned staging buffer, transparent huge pages, and pinned-per-chunk arrays."""
import mmap
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

N = 1 << 24  # u64 values = 128 MB
x = torch.empty(N, dtype=torch.uint64, device="cuda")
stage = torch.empty(N, dtype=torch.uint64, pin_memory=True)
stage.copy_(x)
src = stage.numpy()
print("cpus", os.cpu_count(), "thp", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
pool = ThreadPoolExecutor(16)


def par_copy(dst, src, nt):
    step = -(-dst.size // nt)
    list(pool.map(lambda i: np.copyto(dst[i * step:(i + 1) * step], src[i * step:(i + 1) * step]), range(nt)))


def fresh_np():
    return np.empty(N, dtype=np.uint64)


def fresh_thp():
    m = mmap.mmap(-1, N * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=np.uint64)


def t(label, fn, reps=8):
    fn()
    s = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = (time.perf_counter() - s) / reps
    print(f"{label:40s} {N * 8 / dt / 1e9:6.1f} GB/s")


t("fresh np, 1 thread", lambda: np.copyto(fresh_np(), src))
for nt in (4, 8, 16):
    t(f"fresh np, {nt} threads", lambda: par_copy(fresh_np(), src, nt))
t("fresh thp, 1 thread", lambda: np.copyto(fresh_thp(), src))
for nt in (4, 8, 16):
    t(f"fresh thp, {nt} threads", lambda: par_copy(fresh_thp(), src, nt))
def pinned_chunk():
    h = torch.empty(N, dtype=torch.uint64, pin_memory=True)
    h.copy_(x)
    return h.numpy()
t("pinned per chunk (cached allocator)", pinned_chunk)

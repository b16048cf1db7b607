"""Fresh host arrays (the reference's chunk ownership, generators.py:482):
first-touch copy rate of a pinned 256 MB staging buffer into a new numpy
array, plain vs madvise(MADV_HUGEPAGE), 1 and 16 threads.  Prints the THP
mode of the box and one line per variant."""
import ctypes
import mmap
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

N = 1 << 25  # uint64 values (256 MB)
MADV_HUGEPAGE = 14
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]

try:
    print("thp:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
          "| defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
except OSError as e:
    print("thp: n/a", e)

src = torch.empty(N, dtype=torch.uint64, pin_memory=True).numpy()
src[:] = np.arange(N, dtype=np.uint64)
pool = ThreadPoolExecutor(16)


def alloc(kind):
    if kind == "np.empty":
        return np.empty(N, dtype=np.uint64)
    if kind == "np.empty+madvise":
        a = np.empty(N, dtype=np.uint64)
        p = a.ctypes.data
        lo = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
        hi = (p + a.nbytes) & ~((2 << 20) - 1)
        if hi > lo:
            libc.madvise(lo, hi - lo, MADV_HUGEPAGE)
        return a
    m = mmap.mmap(-1, N * 8 + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    off = (-base) % (2 << 20)
    libc.madvise(base + off, N * 8, MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=np.uint64, count=N, offset=off)


def copy(dst, nt):
    if nt == 1:
        np.copyto(dst, src)
        return
    step = -(-N // nt)
    list(pool.map(lambda i: np.copyto(dst[i * step:(i + 1) * step], src[i * step:(i + 1) * step]), range(nt)))


for kind in ["np.empty", "np.empty+madvise", "mmap+madvise"]:
    for nt in (1, 16):
        best = 0.0
        for _ in range(4):
            t = time.perf_counter()
            d = alloc(kind)
            copy(d, nt)
            dt = time.perf_counter() - t
            assert d[N - 1] == N - 1
            best = max(best, N * 8 / dt / 1e9)
            del d
        print(f"{kind:18s} threads={nt:2d}  {best:6.1f} GB/s", flush=True)

"""A/B the headline fill of two library builds on one box (sustained, 300
steps each, alternating): plain ctypes, so older builds whose C ABI lacks
newer symbols can be compared.  usage: python profiles/ab_fill_lib.py a.so b.so"""
import ctypes
import sys

import torch

N, T, K = 1 << 20, 1024, 4


def run(path, steps=300):
    L = ctypes.CDLL(path)
    gid = L.slp_generator_id(b"xoshiro256starstar")
    u64 = ctypes.c_uint64
    base = (u64 * 4)(0xbdd732262feb6e95, 0x28efe333b266f103, 0x47526757130f9f52, 0x581ce1ff0e4ae394)
    steps_w = (u64 * 3)(0, 0, 1)  # 2^128
    S = torch.empty((K, N), dtype=torch.uint64, device="cuda")
    out = torch.empty((N, T), dtype=torch.uint64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    L.slp_init_substreams.argtypes = [ctypes.c_int, ctypes.POINTER(u64), u64, ctypes.POINTER(u64), ctypes.c_int,
                                      ctypes.c_void_p, u64, u64, ctypes.c_void_p]
    L.slp_fill.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, u64, u64, u64, ctypes.c_int, ctypes.c_int,
                           ctypes.c_void_p, u64, ctypes.c_void_p]
    assert L.slp_init_substreams(gid, base, 1, steps_w, 3, ctypes.c_void_p(S.data_ptr()), N, N, st) == 0
    sp, op = ctypes.c_void_p(S.data_ptr()), ctypes.c_void_p(out.data_ptr())
    L.slp_last_error.restype = ctypes.c_char_p
    for _ in range(10):
        rc = L.slp_fill(gid, sp, sp, N, N, T, 0, 0, op, T, st)
        assert rc == 0, (path, rc, L.slp_last_error())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        L.slp_fill(gid, sp, sp, N, N, T, 0, 0, op, T, st)
    e1.record()
    e1.synchronize()
    return N * T * steps / (e0.elapsed_time(e1) / 1e3)


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        print(sys.argv[2], "%.4g outputs/s" % run(sys.argv[2]), flush=True)
    else:
        import subprocess

        # one process per library: two builds of the same kernels in one
        # process can collide (their launches then fail with invalid argument)
        for rep in range(3):
            for p in sys.argv[1:]:
                subprocess.run([sys.executable, __file__, "--one", p], check=True)

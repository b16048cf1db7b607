"""Interleaved A/B of (library build, store-pacing target) on the config-2
fill: every configuration runs `--launches` back-to-back 8 GiB launches per
round, rounds alternate through all configurations `--rounds` times, and the
median per configuration is reported, so box drift (power cap, heat) hits
every configuration alike.  Plain ctypes; one worker process per build.

  python profiles/ab_pace.py --cfg main:0 --cfg main:6400 --cfg variants/libslp_w14.so:6400 ...
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAIN = os.path.join(ROOT, "paper_1805_01407_b200", "_lib", "libslp_b200.so")
CASES = {  # generator, substreams, T, out kind (SLP_OUT_*: 0 native, 2 f64, 3 f32), element dtype
    "c2": ("xoshiro256starstar", 1 << 20, 1024, 0, torch.uint64, 4, 64),
    "c2f64": ("xoshiro256starstar", 1 << 20, 1024, 2, torch.float64, 4, 64),
    "c3": ("xoroshiro128plus", 1 << 20, 1024, 2, torch.float64, 2, 64),
    "c4": ("xoshiro128starstar", 1 << 21, 1024, 3, torch.float32, 4, 32),
    "x1024": ("xoroshiro1024plusplus", 1 << 20, 1024, 0, torch.uint64, 16, 64),
}


class Lib:
    def __init__(self, path):
        self.L = L = ctypes.CDLL(path)
        u64 = ctypes.c_uint64
        L.slp_init_substreams.argtypes = [ctypes.c_int, ctypes.POINTER(u64), u64, ctypes.POINTER(u64), ctypes.c_int,
                                          ctypes.c_void_p, u64, u64, ctypes.c_void_p]
        L.slp_fill.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, u64, u64, u64, ctypes.c_int,
                               ctypes.c_int, ctypes.c_void_p, u64, ctypes.c_void_p]
        L.slp_set_fill_pace.argtypes = [ctypes.c_int]
        L.slp_last_error.restype = ctypes.c_char_p


def worker(path, case, conn, env=None):
    """One library build per process (two statically linked CUDA runtimes in
    one process fail to launch); runs `launches` fills per request."""
    os.environ.update(env or {})
    gen, n, T, ok, dt, k, w = CASES[case]
    L = Lib(path).L
    wdt = torch.uint64 if w == 64 else torch.uint32
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    out = torch.empty((n, T), dtype=dt, device="cuda")
    S = torch.empty((k, n), dtype=wdt, device="cuda")
    u64 = ctypes.c_uint64
    gid = L.slp_generator_id(gen.encode())
    sys.path.insert(0, ROOT)
    from paper_1805_01407_b200 import generators as G

    base = (u64 * 16)(*G.seed_state(G.get_spec(gen), 42))
    steps_w = (u64 * 3)(0, 0, 1) if w == 64 else (u64 * 2)(0, 1)  # stride 2^128 (w=32: 2^64)
    assert L.slp_init_substreams(gid, base, 1, steps_w, len(steps_w), ctypes.c_void_p(S.data_ptr()), n, n, sp) == 0
    Sp, Op = ctypes.c_void_p(S.data_ptr()), ctypes.c_void_p(out.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    conn.send(out.numel() * out.element_size())
    while True:
        msg = conn.recv()
        if msg is None:
            break
        pace, launches = msg
        L.slp_set_fill_pace(pace)
        e0.record()
        for _ in range(launches):
            rc = L.slp_fill(gid, Sp, Sp, n, n, T, ok, 0, Op, T, sp)
            assert rc == 0, (path, rc, L.slp_last_error())
        e1.record()
        e1.synchronize()
        conn.send(e0.elapsed_time(e1) / launches)


def main():
    import multiprocessing as mp

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", action="append", required=True,
                    help="lib:pace_gbps[:burst] (lib 'main' = the in-tree build; burst -> SLP_FILL_PACE_BURST)")
    ap.add_argument("--case", default="c2")
    ap.add_argument("--launches", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=8)
    a = ap.parse_args()
    ctx = mp.get_context("spawn")
    conns, procs, cfgs = {}, [], []
    for c in a.cfg:
        parts = c.split(":")
        path, pace = parts[0], int(parts[1])
        burst = parts[2] if len(parts) > 2 else "1"
        path = MAIN if path == "main" else os.path.join(ROOT, path) if not os.path.isabs(path) else path
        key = (path, burst)
        if key not in conns:
            here, there = ctx.Pipe()
            pr = ctx.Process(target=worker, args=(path, a.case, there, {"SLP_FILL_PACE_BURST": burst}))
            pr.start()
            procs.append(pr)
            conns[key] = here
        cfgs.append((key, pace))
    nbytes = [c.recv() for c in conns.values()][0]
    res = {i: [] for i in range(len(cfgs))}

    def run(i, launches):
        key, pace = cfgs[i]
        conns[key].send((pace, launches))
        return conns[key].recv()

    for i in range(len(cfgs)):
        run(i, 3)
    for r in range(a.rounds):
        order = list(range(len(cfgs)))
        if r % 2:
            order.reverse()
        for i in order:
            res[i].append(run(i, a.launches))
    for c in conns.values():
        c.send(None)
    for pr in procs:
        pr.join()
    for i, ((path, burst), pace) in enumerate(cfgs):
        med = statistics.median(res[i])
        print(json.dumps({"case": a.case, "lib": os.path.relpath(path, ROOT), "pace_gbps": pace, "burst": int(burst),
                          "ms_median": round(med, 4), "GBps": round(nbytes / med / 1e6, 1),
                          "ms_min": round(min(res[i]), 4), "ms_max": round(max(res[i]), 4)}), flush=True)


if __name__ == "__main__":
    main()

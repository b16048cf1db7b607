#!/usr/bin/env python
"""Headline benchmark: BASELINE.json config 2 with xoshiro256** —
2^20 substreams (stream i = seed 42 jumped i * 2^128), 1024 uint64 outputs
each, stored stream-major to HBM (8 GiB per step) by kernel K2 (TMA stores).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over the batch: every substream emits its
next 1024 outputs (states resident in HBM, advanced in place).  The output
(8 GiB) is far larger than L2 (126 MB), so no L2 flush is needed between
steps.  Multi-GPU (torchrun): rank r generates long-jump block r (substreams
seed * M^(r*2^192 + i*2^128)); there is no data-path collective (weak scaling);
timing is the max over ranks of CUDA-event time.  ``--gpus N`` without a
torchrun environment re-launches itself under ``torch.distributed.run`` with N
ranks (one per GPU, NCCL).  ``--impl reference`` times the UNMODIFIED reference
package (``baseline/_ref/slprng``, its own LanedStream set-up + VecStepper /
apply_vec loop, oracle/ref_baseline.py) on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GEN = "xoshiro256starstar"
SEED = 42
N_STREAMS = 1 << 20
T = 1024
METRIC = "xoshiro256** 64-bit outputs/s"
UNIT = "outputs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the fused-mode (K4) roofline, the config-5 job and the f64 store line")
    return ap.parse_args()


def config(world):
    return {"workload": "BASELINE config 2: xoshiro256** 2^20 substreams x 1024 u64, store mode (8 GiB/step/GPU)",
            "generator": GEN, "seed": SEED, "substreams_per_gpu": N_STREAMS, "outputs_per_substream": T,
            "layout": "stream-major [substream][position]", "store_path": "TMA bulk tensor store (K2)",
            "l2": "output 8 GiB/step >> 126 MB L2; no flush needed",
            "partition": "rank r = long-jump block r (seed*M^(r*2^192))", "world_size": world}


# ---------------------------------------------------------------- clocks (NVML)


class ClockSampler:
    """Samples SM clock and throttle reasons every 10 ms in a thread."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self.samples = []
        self.reasons = 0
        self._stop = threading.Event()

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.01)

    def start(self):
        self.samples, self.reasons = [], 0
        self._stop.clear()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self):
        self._stop.set()
        self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------- helpers


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_traffic(kernel_tag):
    """dram read+write bytes per launch of the fill kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel_tag, {}).get("dram_bytes_per_launch")
    except OSError:
        return None


FUSED_PIPES = "round2_fused_pipes.json"  # profiles/make_fused_pipes.py on the current build


def fused_pipes():
    try:
        with open(os.path.join(ROOT, "profiles", FUSED_PIPES)) as f:
            return json.load(f)
    except OSError:
        return {}


def golden_checksum(key):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "checksums_big.json")) as f:
            return json.load(f).get(key, {})
    except OSError:
        return {}


def cpu_baseline():
    """The stock reference (baseline/_ref/slprng) on the host cores: config 2's
    exact partition (2^20 substreams, resident states), one checked warm-up
    step + 3 timed steps; then the same on one core over 2^15 substreams."""
    from oracle.ref_baseline import ReferenceArm

    g = golden_checksum(f"c2/{GEN}")
    arm = ReferenceArm(GEN, SEED, N_STREAMS, T, setup_each_step=True)
    try:
        _, _, s0, x0 = arm.step(checksum=True)
        secs, gen = [], []
        for _ in range(3):
            secs.append(arm.step()[1])
            gen.append(arm.last_generate_s)
    finally:
        arm.close()
    res = {"value": 3 * N_STREAMS * T / sum(secs), "unit": UNIT, "cores": arm.procs, "kind": "reference",
           "sample": f"3 steps x config 2 from the seed (2^20 substreams x {T} outputs), stock slprng from "
                     f"baseline/_ref: Generator.jump + LanedStream set-up, then apply_vec + VecStepper.step "
                     f"into a (T, 2^14) buffer per chunk, {arm.procs} worker processes",
           "matches_reference": bool(g) and (hex(s0), hex(x0)) == (g["sum"], g["xor"]),
           "value_resident_states": 3 * N_STREAMS * T / sum(gen)}
    one = ReferenceArm(GEN, SEED, 1 << 15, T, procs=1, setup_each_step=True)
    try:
        one.step()
        n1, dt1 = one.step()
    finally:
        one.close()
    res["value_1core"] = n1 / dt1
    res["sample_1core"] = f"1 process x 2^15 substreams x {T} outputs from the seed (stock slprng)"
    return res


# ---------------------------------------------------------------- our arm


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1805_01407_b200 as P
    from paper_1805_01407_b200 import device as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SLP_BENCH_SHARE_GPU=1 (flow check of the N > 1 path on a one-GPU box, not a
    # measurement): every rank uses cuda:0 and gloo carries the collectives
    share = os.environ.get("SLP_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    elif world > torch.cuda.device_count():
        sys.exit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPUs")
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    spec = P.get_spec(GEN)
    k = spec.kind.k

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # substream init (K1), timed separately (setup; not in the step)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    D.Substreams.from_seed(spec, SEED, N_STREAMS, first_block=rank)  # plan + poly upload (host, once)
    torch.cuda.synchronize()
    t0.record()
    sub = D.Substreams.from_seed(spec, SEED, N_STREAMS, first_block=rank)
    t1.record()
    torch.cuda.synchronize()
    init_ms = t0.elapsed_time(t1)

    out = torch.empty((N_STREAMS, T), dtype=torch.uint64, device=dev)

    def write_only_sweep():
        # live write-only ceiling of this GPU: a forward-sweep fill of the same
        # 8 GiB tensor (torch fill_, measurement reference only, outside the timed region)
        for _ in range(2):
            out.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            out.fill_(1)
        e1.record()
        torch.cuda.synchronize()
        return N_STREAMS * T * 8 / (e0.elapsed_time(e1) / 10 / 1e3) / 1e9

    write_only_before = write_only_sweep()  # cool GPU (before the sustained steps)
    for _ in range(args.warmup):
        sub.fill(T, out=out)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(args.steps):
        sub.fill(T, out=out)
    end.record()
    clocks.sample()
    torch.cuda.synchronize()
    clocks.stop()
    barrier()
    torch.cuda.synchronize()
    ms_local = start.elapsed_time(end)
    ms = max_over_ranks(ms_local)

    write_only_after = write_only_sweep()  # same GPU state as the timed steps
    write_only_gbs = max(write_only_before, write_only_after)
    outputs_per_step = N_STREAMS * T * world
    value = outputs_per_step * args.steps / (ms / 1e3)

    # roofline of the dominant (only) kernel of the step: k_fill<xoshiro256**, native, TMA>
    launch_ms = ms_local / args.steps
    alg_bytes = N_STREAMS * T * 8 + 2 * N_STREAMS * k * 8
    peaks, src = measured_peaks()
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    traffic = ncu_traffic("k_fill_xoshiro256starstar_u64_tma")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
                "peak_source": f"{src} (MEASURED_PEAKS.json hbm_gbs: copy read+write, burst)",
                "alg_bytes_per_launch": alg_bytes,
                "alg_bytes_per_unit": "8 B per u64 output + 64 B state read/write per substream per launch",
                "kernel": "k_fill<xoshiro256**, u64, TMA>", "launch_ms": round(launch_ms, 4),
                "frac_of_8TBps_spec": round(achieved / 8000.0, 4),
                "write_only_ceiling_gbs": round(write_only_gbs, 1),
                "frac_of_write_only_ceiling": round(achieved / write_only_gbs, 4),
                "write_only_before_after_gbs": [round(write_only_before, 1), round(write_only_after, 1)],
                "write_only_note": "forward-sweep fill_ of the same 8 GiB tensor, measured live on this GPU before "
                                   "the warm-up and after the timed steps; the ceiling is the larger",
                "frac_of_write_pattern_ceiling": round(achieved / 6708.0, 4),
                "write_pattern_ceiling_note": "6708 GB/s = best TMA-only store of the same stream-major pattern and "
                                              "geometry (1 KiB row pieces, 7 warps x 1 buffer, no generation) under "
                                              "store pacing; 6106 unpaced (profiles/round2_pacing.md)",
                "store_pacing_gbps": D.set_fill_pace(None)}

    # e2e: public API from the seed to HOST memory, every step: substream init
    # (H2D: the base state, k words) + fill + D2H of all outputs (pinned), overlapped
    e2e = None
    host, pin_err = None, ""
    if args.e2e_steps > 0:
        try:  # 8 GiB pinned per rank; every rank must succeed or all skip (no hang in collectives)
            host = torch.empty((N_STREAMS, T), dtype=torch.uint64, pin_memory=True)
        except Exception as e:  # noqa: BLE001
            pin_err = f"pinned host buffer allocation failed: {e}"[:200]
        ok = 1.0 if host is not None else 0.0
        if world > 1:
            t_ok = torch.tensor([ok], dtype=torch.float64, device=dev)
            dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
            ok = float(t_ok.item())
        if ok < 1.0:
            e2e = {"error": pin_err or "pinned allocation failed on another rank"}
            host = None
    if host is not None:
        bufs = [torch.empty((1 << 15, T), dtype=torch.uint64, device=dev) for _ in range(2)]
        del out
        # two untimed passes: the first DMA into freshly pinned pages runs ~15%
        # slower (profiles/round2_e2e_steps.jsonl)
        for i in range(args.e2e_steps + 2):
            if i == 2:
                barrier()
                torch.cuda.synchronize()
                t_start = time.perf_counter()
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
            s2 = D.Substreams.from_seed(spec, SEED, N_STREAMS, first_block=rank)
            D.fill_to_host(spec, s2.states, T, host, _bufs=bufs)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        torch.cuda.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1))
        wall = time.perf_counter() - t_start
        e2e = {"value": outputs_per_step * args.e2e_steps / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": k * 8, "d2h_bytes_per_step": N_STREAMS * T * 8,
               "api": "Substreams.from_seed + device.fill_to_host (pinned host, D2H overlapped)",
               "ms_per_step": round(e_ms / args.e2e_steps, 3), "wall_s": round(wall, 3)}
        del host, bufs

    # the same API call when the consumer is on the GPU: per step the base state
    # goes in (kernel parameters), substreams are initialised (K1) and filled
    # (K2) into a device tensor, and one output word is read back as the result
    e2e_dev = None
    if args.e2e_steps > 0:
        outd = torch.empty((N_STREAMS, T), dtype=torch.uint64, device=dev)
        res_host = torch.empty(1, dtype=torch.uint64, pin_memory=True)
        for i in range(args.e2e_steps + 3):
            if i == 3:
                barrier()
                torch.cuda.synchronize()
                f0 = torch.cuda.Event(enable_timing=True)
                f0.record()
            s3 = D.Substreams.from_seed(spec, SEED, N_STREAMS, first_block=rank)
            s3.fill(T, out=outd)
            res_host.copy_(outd[-1, -1:], non_blocking=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f1.record()
        torch.cuda.synchronize()
        f_ms = max_over_ranks(f0.elapsed_time(f1))
        e2e_dev = {"value": outputs_per_step * args.e2e_steps / (f_ms / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": k * 8, "d2h_bytes_per_step": 8,
                   "api": "Substreams.from_seed + Substreams.fill (device tensor), init included",
                   "ms_per_step": round(f_ms / args.e2e_steps, 4)}
        del outd

    # the reference's own bulk API, drop-in: output_stream -> fresh numpy chunks
    # (single stream, 2^16 lanes x 1024 per superbatch, 2^30 values)
    e2e_os = None
    if args.e2e_steps > 0:
        total = 1 << 30
        # warm-up stream: init plans and the process's pool of page-locked
        # chunk buffers (pinning 3 x 512 MB once per process)
        for c in P.output_stream(spec, SEED + 1, 1 << 28, lanes=1 << 16, lane_len=1024):
            pass  # a consumer holding one chunk while the next is produced: 3 buffers
        t_os = time.perf_counter()
        got = 0
        for c in P.output_stream(spec, SEED, total, lanes=1 << 16, lane_len=1024):
            got += c.size
        dt_os = time.perf_counter() - t_os
        del c
        e2e_os = {"value": got / dt_os, "unit": "values/s",
                  "api": "output_stream(spec, 42, 2^30, lanes=2^16, lane_len=1024) from the seed: numpy uint64 "
                         "chunks owned by the caller (DMA into pooled page-locked buffers, recycled when dropped)",
                  "wall_s": round(dt_os, 3)}

    extra = {}
    if not args.no_extra:
        extra = run_extra(spec, dev, rank, world)

    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline()
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded, SplitMix64)",
                "config": config(world), "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
                "e2e_device_resident": e2e_dev, "e2e_output_stream": e2e_os,
                "clocks": clocks.summary(), "gpu_launches": args.steps,
                "init_ms_2^20_substreams": round(init_ms, 3)}
        line.update(extra)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_extra(spec, dev, rank, world):
    """Fused mode (K4) with its INT roofline on the same substreams, the
    config-5 job (sharded over the ranks, one collective) and the f64 store."""
    import torch

    import paper_1805_01407_b200 as P
    from paper_1805_01407_b200 import device as D

    res = {}
    sub = D.Substreams.from_seed(spec, SEED, N_STREAMS, first_block=rank)
    raw = torch.empty(48, dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    for label, kw in (("fused_int", dict(exact=False)), ("fused_exact", dict(exact=True)),
                      ("fused_exact_f64", dict(exact=True, f64=True))):
        for _ in range(3):
            sub.checksum_async(T, result=raw, **kw)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            sub.checksum_async(T, result=raw, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[label] = {"outputs_per_s": N_STREAMS * T / (ms / 1e3), "ms_per_step": ms}
        # INT roofline of K4: ALU-pipe SASS per output (committed ncu pipe counts)
        # x outputs/s against the measured ALU-pipe peak (profiles/int_peak.cu)
        pipes = fused_pipes().get({"fused_int": "sum_xor", "fused_exact": "exact",
                                   "fused_exact_f64": "exact_f64"}[label])
        if pipes:
            peak = fused_pipes()["int_peaks"]["alu_warp_inst_per_s"]
            ach = res[label]["outputs_per_s"] * pipes["alu_sass_per_output"] / 32
            res[label]["roofline"] = {"bound": "int (ALU pipe)", "achieved": ach, "peak": peak,
                                      "unit": "warp-inst/s", "frac": round(ach / peak, 4),
                                      "alu_sass_per_output": round(pipes["alu_sass_per_output"], 3),
                                      "source": "profiles/" + FUSED_PIPES}
    # config 5 whole job: 2^34 outputs = 8 long-jump blocks x 2^18 substreams x 2^13,
    # blocks b == rank (mod world), fused exact checksum per GPU, one all_gather
    import torch.distributed as dist

    from paper_1805_01407_b200.multigpu import sharded_checksum

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # config 5 as a whole job: 2^34 outputs = 8 long-jump blocks x 2^18 substreams
    # x 2^13, blocks b == rank (mod world), fused exact checksum per GPU, ONE
    # all_gather of the 64-byte per-rank records (NCCL under torchrun), then
    # the fold; job time = max over ranks of the barrier-to-result wall time
    c5 = {}
    for name in ("xoshiro512starstar", "xoroshiro1024plusplus"):
        s5 = P.get_spec(name)
        sharded_checksum(s5, 42, 8, 1 << 18, 1 << 4, rank=rank, world=world)  # warm host plans + collective
        sync_all()
        t0 = time.perf_counter()
        total, parts = sharded_checksum(s5, 42, 8, 1 << 18, 1 << 13, rank=rank, world=world)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        g = golden_checksum(f"c5/{name}")
        c5[name] = {"job_s": round(dt, 4), "outputs_per_s": (1 << 34) / dt, "ranks": world,
                    "blocks_per_rank": [len(range(r, 8, world)) for r in range(world)],
                    "collective": ("all_gather (" + dist.get_backend() + ")") if world > 1 else "none (1 rank)",
                    "matches_reference": bool(g) and hex(total.sum) == g["sum"] and hex(total.xor) == g["xor"]
                    and hex(total.mant) == g["mant"], "sum": hex(total.sum), "xor": hex(total.xor)}
    res["config5_job"] = c5
    out = torch.empty((N_STREAMS, T), dtype=torch.float64, device=dev)
    sub.fill(T, out=out, kind="f64")
    e0.record()
    for _ in range(20):
        sub.fill(T, out=out, kind="f64")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res["store_f64"] = {"outputs_per_s": N_STREAMS * T / (ms / 1e3), "ms_per_step": ms}
    return res


# ---------------------------------------------------------------- reference arm


def run_reference(args):
    """The UNMODIFIED reference (baseline/_ref/slprng) on this box's host
    cores, same metric/config/unit as our arm; rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.ref_baseline import ReferenceArm

    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    g = golden_checksum(f"c2/{GEN}")
    arm = ReferenceArm(GEN, SEED, N_STREAMS, T, setup_each_step=True)
    try:
        # warm-up: the first step from the fresh set-up is config 2 itself -> checked
        _, _, s0, x0 = arm.step(checksum=True)
        for _ in range(max(0, args.warmup - 1)):
            arm.step()
        secs, gen = [], []
        for _ in range(args.steps):
            secs.append(arm.step()[1])
            gen.append(arm.last_generate_s)
    finally:
        arm.close()
    tot = N_STREAMS * T * args.steps
    value = tot / sum(secs)
    sample = (f"each step: config 2 from the seed (2^20 substreams x {T} outputs), stock slprng from "
              f"baseline/_ref: Generator.jump + LanedStream(lane_len=2^128) set-up per 2^14-lane chunk, "
              f"then T x (ScramblerSpec.apply_vec, VecStepper.step) into a (T, L) buffer, "
              f"{arm.procs} worker processes")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(secs) / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded, SplitMix64)", "config": config(world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": arm.procs, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "matches_reference": bool(g) and (hex(s0), hex(x0)) == (g["sum"], g["xor"]),
            "setup_s": round(arm.init_wall_s, 3),
            # the same steps without the set-up (states resident, as in our arm's kernel step)
            "value_resident_states": tot / sum(gen),
            "note": "the GPU arm's world x 2^20 substreams are not replicated here: one host, "
                    "rank 0 runs the per-GPU workload once"}
    print(json.dumps(line))


def relaunch_if_needed(args):
    """--gpus N > 1 without a torchrun environment: re-exec under
    torch.distributed.run (one rank per GPU); with one, require WORLD_SIZE == N."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to measure "
                     f"a different GPU count than requested")
        return
    if args.gpus <= 1:
        return
    import socket
    import subprocess

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    relaunch_if_needed(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

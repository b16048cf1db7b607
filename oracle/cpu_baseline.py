"""CPU baseline — TEST/BENCH INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg
and ``bench.py --impl reference``).

Times the reference's own CPU algorithm for the config-2 path, restated in
oracle/oracle.py (numpy lanes: lane set-up by polynomial-jump doubling,
generators.py:443-459; then T x (ScramblerSpec.apply_vec, VecStepper.step),
scramblers.py:97-127, engines.py:318-361), on every host core: each worker
process owns a contiguous slice of substreams, exactly the recipe of
BASELINE.md section 2 / SURVEY.md section 8(d).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import oracle as O


def _worker(args):
    name, seed, c0, c1, T = args
    n = O.SPECS[name][1] * O.SPECS[name][2]
    J = 1 << (n // 2)
    flat = O.seed_flat(name, seed)
    if c0:
        flat = O.jump(name, flat, O.jump_poly(name, c0 * J))
    S = O.lane_states(name, flat, c1 - c0, J)
    t0 = time.perf_counter()
    buf = np.empty((T, c1 - c0), dtype=np.uint64)
    for t in range(T):
        buf[t] = O.vec_scramble(name, S)
        S = O.vec_step(name, S)
    acc = int(np.bitwise_xor.reduce(buf.reshape(-1)))
    return acc, time.perf_counter() - t0


class CpuBaseline:
    """A process pool over all host cores running the reference algorithm."""

    def __init__(self, name="xoshiro256starstar", seed=42, T=1024, procs=None):
        self.name, self.seed, self.T = name, seed, T
        self.procs = procs or os.cpu_count() or 1
        self.pool = mp.get_context("fork").Pool(self.procs)
        # warm the char-poly / jump caches in the workers
        self.pool.map(_worker, [(name, seed, 0, 2, 2)] * self.procs)
        self.next_stream = 0

    def step(self, lanes_per_worker: int):
        """One bounded sample: procs x lanes_per_worker substreams x T outputs.
        Returns (outputs, seconds)."""
        tasks = []
        for _ in range(self.procs):
            c0 = self.next_stream
            tasks.append((self.name, self.seed, c0, c0 + lanes_per_worker, self.T))
            self.next_stream += lanes_per_worker
        t0 = time.perf_counter()
        self.pool.map(_worker, tasks, chunksize=1)
        dt = time.perf_counter() - t0
        return self.procs * lanes_per_worker * self.T, dt

    def calibrate(self, target_s: float) -> int:
        """lanes per worker giving roughly target_s per step."""
        lanes = 2048
        n, dt = self.step(lanes)
        per_lane = dt / lanes
        return max(2048, min(1 << 17, int(target_s / per_lane)))

    def close(self):
        self.pool.close()
        self.pool.join()

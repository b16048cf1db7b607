"""Stock-reference CPU arm — BENCH INFRASTRUCTURE ONLY (bench.py's
``cpu_baseline`` leg and ``bench.py --impl reference``).

Runs the UNMODIFIED reference package ``slprng`` (installed once into
``baseline/_ref`` by ``__graft_entry__.build()`` with ``pip install --target``;
git-ignored, travels to the GPU box) through its own public API on every host
core, on BASELINE config 2's exact partition:

* substreams [0, 2^20) of seed 42 (stream i = seed * M^(i * 2^128)) are split
  into contiguous slices, one per worker process;
* each slice is set up with the reference's own calls, in chunks of 2^14
  lanes (the chunk size that ran fastest per core, profiles/round2_ref_vs_port.md):
  ``g = Generator.from_seed(spec, 42); g.jump(compute_jump_poly(spec, c0 << 128))``
  then ``LanedStream(spec, generator=g, lanes=c1 - c0, lane_len=2^128).S``
  (generators.py:315-334, 397-402, 435-463);
* one step = every substream emits its next T = 1024 outputs into a (T, L)
  buffer (the reference's own ``chunks`` loop body, generators.py:476-480):
  ``buf[t] = spec.scrambler.apply_vec(st.word(S, i), st.word(S, j), w);
  st.step(S)`` (scramblers.py:97-127, engines.py:318-361).  With
  ``setup_each_step`` (bench.py's reference arm) the stock set-up above is
  redone inside every step, from the seed, as the GPU arm's e2e leg does
  (``Substreams.from_seed`` every step); without it the states stay resident
  in each worker and advance in place (the GPU arm's kernel step).

The first step from a fresh set-up is config 2 itself, so its wrapping sum
and xor (reduced outside the timed steps) are checked against the golden
checksums in tests/golden/checksums_big.json.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
CHUNK = 1 << 14


def import_reference():
    """The stock slprng from baseline/_ref (never the in-tree package)."""
    if not os.path.isdir(os.path.join(REF_DIR, "slprng")):
        raise ImportError(f"reference not installed at {REF_DIR} (run __graft_entry__.build())")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import slprng
    import slprng.engines  # noqa: F401  (VecStepper lives here in the reference)

    if not os.path.abspath(slprng.__file__).startswith(REF_DIR):
        raise ImportError(f"slprng resolved to {slprng.__file__}, not {REF_DIR}")
    return slprng


def _worker(conn, name, seed, s0, s1, T, chunk, setup_each_step):
    R = import_reference()
    spec = R.get_spec(name)
    n = spec.kind.n
    J = 1 << (n // 2)
    sc = spec.scrambler
    w = spec.kind.w

    def setup():
        lanes = []
        for c0 in range(s0, s1, chunk):
            c1 = min(s1, c0 + chunk)
            g = R.Generator.from_seed(spec, seed)
            if c0:
                g.jump(R.compute_jump_poly(spec, c0 * J))
            ls = R.LanedStream(spec, generator=g, lanes=c1 - c0, lane_len=J)
            lanes.append((ls.S, ls.stepper))
        return lanes

    t0 = time.perf_counter()
    lanes = setup()
    init_s = time.perf_counter() - t0
    buf = np.empty((T, min(chunk, max(1, s1 - s0))), dtype=np.uint64)
    conn.send(("ready", init_s))
    first = True
    while True:
        cmd = conn.recv()
        if cmd == "stop":
            break
        checksum = cmd == "step+checksum"
        acc_sum, acc_xor = 0, 0
        t0 = time.perf_counter()
        setup_s = 0.0
        if setup_each_step and not first:  # from the seed again: the stock lane set-up is part of the step
            lanes = setup()
            setup_s = time.perf_counter() - t0
        first = False
        for S, st in lanes:
            L = S.shape[1]
            b = buf[:, :L]
            for t in range(T):
                xi = st.word(S, sc.word_i)
                xj = st.word(S, sc.word_j) if sc.word_j is not None else None
                b[t] = sc.apply_vec(xi, xj, w)
                st.step(S)
            if checksum:  # only on the first (untimed, warm-up) step
                acc_sum = (acc_sum + int(np.add.reduce(b, axis=None, dtype=np.uint64))) & ((1 << 64) - 1)
                acc_xor ^= int(np.bitwise_xor.reduce(b, axis=None))
        conn.send(("done", time.perf_counter() - t0, acc_sum, acc_xor, setup_s))


class ReferenceArm:
    """Worker processes over all host cores, each owning a contiguous slice of
    the substreams with resident states (set up by the stock reference)."""

    def __init__(self, name="xoshiro256starstar", seed=42, n_streams=1 << 20, T=1024, procs=None,
                 chunk=CHUNK, setup_each_step=False):
        import_reference()  # fail here, in the parent, if it is missing
        self.name, self.seed, self.n, self.T = name, seed, n_streams, T
        self.procs = max(1, min(procs or os.cpu_count() or 1, n_streams))
        ctx = mp.get_context("fork")  # children never touch CUDA
        self.conns, self.ps = [], []
        per = -(-n_streams // self.procs)
        t0 = time.perf_counter()
        for p in range(self.procs):
            s0, s1 = p * per, min(n_streams, (p + 1) * per)
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_worker, args=(b, name, seed, s0, s1, T, chunk, setup_each_step), daemon=True)
            pr.start()
            self.conns.append(a)
            self.ps.append(pr)
        inits = [c.recv()[1] for c in self.conns]
        self.init_wall_s = time.perf_counter() - t0
        self.init_worker_s = max(inits)
        self.steps_done = 0

    def step(self, checksum=False):
        """One step (T outputs per substream on every worker).  Returns
        (outputs, wall seconds[, wrapping sum, xor]); ``last_generate_s`` is
        the slowest worker's step time without its set-up."""
        cmd = "step+checksum" if checksum else "step"
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(cmd)
        res = [c.recv() for c in self.conns]
        wall = time.perf_counter() - t0
        self.last_generate_s = max(r[1] - r[4] for r in res)
        self.steps_done += 1
        if checksum:
            s, x = 0, 0
            for r in res:
                s = (s + r[2]) & ((1 << 64) - 1)
                x ^= r[3]
            return self.n * self.T, max(r[1] for r in res), s, x
        return self.n * self.T, wall

    def close(self):
        for c in self.conns:
            try:
                c.send("stop")
            except (BrokenPipeError, OSError):
                pass
        for p in self.ps:
            p.join(timeout=10)

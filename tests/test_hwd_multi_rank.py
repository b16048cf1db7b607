"""Multi-rank HWD host logic on CPU: two gloo ranks each count their slice of
every checkpoint range (CPU oracle counter instead of kernel K6), the
counters are all-reduced, and both ranks must return the reference's report
(tests/golden/hwd.json, produced by the reference itself)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_01407_b200 import hwd

CASE = "xoshiro256starstar/3/60000/byte_limit=1600000,k=4,w=64"
CASE_T = "xoroshiro128plus/5/500000/byte_limit=32000000,k=6,mode=transitional,w=64"


class OracleCounter:
    """Drop-in for hwd._GpuCounter backed by the numpy oracle (test infrastructure)."""

    def __init__(self, spec, seed, cfg, device=None):
        from oracle import oracle as O

        self.O, self.spec, self.seed, self.cfg = O, spec, seed, cfg
        n = 3 ** cfg.k
        self.counts = np.zeros(n, np.uint64)
        self.sums = np.zeros(n, np.uint64)
        self.values = None

    def count(self, c0, c1):
        cfg = self.cfg
        if self.values is None or self.values.size < c1:
            self.values = self.O.hwd_test_values(self.spec.name, self.seed, max(c1, 1 << 16), cfg.split,
                                                 cfg.mode == "transitional", cfg.w)
        c, s = self.O.hwd_counts(self.values, c0, c1, cfg.k, cfg.w, cfg.ell)
        self.counts += c
        self.sums += s

    def totals(self):
        return torch.from_numpy(self.counts.view(np.int64)), torch.from_numpy(self.sums.view(np.int64))


def _expect(G, key):
    d = G("hwd")[key]
    return d, {k: v for k, v in d.items() if k not in ("name", "seed", "checkpoint_start", "config", "ref_seconds")}


def _run(d):
    return hwd.run_generator(d["name"], hwd.HwdConfig(**d["config"]), seed=d["seed"],
                             checkpoint_start=d["checkpoint_start"], _counter_cls=OracleCounter).to_dict()


@pytest.mark.parametrize("key", [CASE, CASE_T])
def test_single_process_oracle_counter_matches_reference(G, key):
    d, want = _expect(G, key)
    assert _run(d) == want


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, d):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(d)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("key", [CASE, CASE_T])
def test_two_ranks_all_reduce_matches_reference(G, key):
    d, want = _expect(G, key)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, d)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == want and res[1] == want

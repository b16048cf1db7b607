"""Multi-GPU host logic on CPU: two gloo ranks partition config-5 style work
by long-jump block (b == rank mod world) and fold their checksums with one
all_gather; the result must equal the single-process checksum, which must
equal the reference's golden value.  Per-rank checksums come from the CPU
oracle (no GPU), so only the partition / collective / fold logic is tested."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1805_01407_b200 as P
from paper_1805_01407_b200.device import Checksum
from paper_1805_01407_b200.multigpu import blocks_for_rank, sharded_checksum


def oracle_compute(spec, seed, blocks, S, T, exact=True):
    from oracle import oracle as O

    name = spec.name
    n = spec.kind.n
    parts = []
    for b in blocks:
        base = O.seed_flat(name, seed)
        if b:
            base = O.jump(name, base, O.jump_poly(name, b << (3 * n // 4)))
        lanes = O.lane_states(name, base, S, 1 << (n // 2))
        outs, _ = O.vec_outputs(name, lanes, T)
        c = O.checksum(outs, spec.kind.w)
        v = outs.reshape(-1)
        exact_sum = int((v >> np.uint64(32)).astype(object).sum()) * (1 << 32) + int(
            (v & np.uint64(0xFFFFFFFF)).astype(object).sum())
        parts.append(Checksum(spec.kind.w, c["sum"], exact_sum, c["xor"], c["mant"], v.size, None))
    if not parts:
        return Checksum(spec.kind.w, 0, 0, 0, 0, 0, None)
    return Checksum.fold(parts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, name, seed, nblocks, S, T):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = P.get_spec(name)
        total, parts = sharded_checksum(spec, seed, nblocks, S, T, rank=rank, world=world, compute=oracle_compute)
        q.put((rank, total.sum, total.xor, total.mant, total.count, [p.count for p in parts]))
    finally:
        dist.destroy_process_group()


def test_blocks_for_rank():
    assert blocks_for_rank(0, 2, 8) == [0, 2, 4, 6]
    assert blocks_for_rank(1, 2, 8) == [1, 3, 5, 7]
    assert blocks_for_rank(3, 8, 8) == [3]
    assert sorted(sum((blocks_for_rank(r, 3, 8) for r in range(3)), [])) == list(range(8))
    with pytest.raises(ValueError):
        blocks_for_rank(2, 2, 8)


@pytest.mark.parametrize("name", ["xoshiro512starstar", "xoroshiro1024plusplus"])
def test_two_rank_gloo_fold_matches_golden(G, name):
    g = G("checksums_small")[f"c5s/{name}"]
    nblocks, S, T = g["blocks"], 64, 256   # a slice of c5s (S 256 -> 64, T 2048 -> 256) for speed
    single, _ = sharded_checksum(P.get_spec(name), g["seed"], nblocks, S, T, compute=oracle_compute)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, name, g["seed"], nblocks, S, T)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, s, x, mant, count, per_rank in res:
        assert (s, x, mant, count) == (single.sum, single.xor, single.mant, single.count)
        assert per_rank == [4 * S * T, 4 * S * T]


def test_fold_full_c5s_matches_golden(G):
    """Block-by-block fold at the golden size equals the reference's checksum."""
    g = G("checksums_small")["c5s/xoshiro512starstar"]
    spec = P.get_spec(g["name"])
    total, _ = sharded_checksum(spec, g["seed"], g["blocks"], g["substreams"], g["T"], compute=oracle_compute)
    assert hex(total.sum) == g["sum"] and hex(total.xor) == g["xor"] and hex(total.mant) == g["mant"]


def test_collective_device_follows_backend(monkeypatch):
    """NCCL rejects CPU tensors: with device=None the all_gather tensor goes to
    the current CUDA device under nccl and stays on the CPU under gloo."""
    import torch

    from paper_1805_01407_b200 import multigpu

    monkeypatch.setattr(dist, "get_backend", lambda group=None: "nccl")
    monkeypatch.setattr(torch.cuda, "current_device", lambda: 3)
    assert multigpu.collective_device() == torch.device("cuda", 3)
    assert multigpu.collective_device(device="cpu") == torch.device("cpu")
    monkeypatch.setattr(dist, "get_backend", lambda group=None: "gloo")
    assert multigpu.collective_device() == torch.device("cpu")
    assert multigpu.collective_device(device="cuda:1") == torch.device("cuda", 1)

"""The multi-rank paths with the REAL device compute: two processes share
the one GPU of this box (their kernels never wait on each other) and talk
over gloo on CPU tensors.  Config-5-style checksums (K1 + K4 per rank, one
all_gather) and HWD (per-rank range slices, one all-reduce of the counters
per checkpoint) must equal the single-process results and the reference's
golden values."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(target, args, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _init(rank, world, port):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _checksum_worker(rank, world, port, q, name, nblocks, S, T):
    _init(rank, world, port)
    try:
        import paper_1805_01407_b200 as P
        from paper_1805_01407_b200.multigpu import sharded_checksum

        total, _ = sharded_checksum(P.get_spec(name), 42, nblocks, S, T, rank=rank, world=world, device="cpu")
        q.put((rank, (hex(total.sum), hex(total.xor), hex(total.mant))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["xoshiro512starstar", "xoroshiro1024plusplus"])
def test_sharded_checksum_two_ranks_on_gpu(G, name):
    g = G("checksums_small")[f"c5s/{name}"]
    res = _run(_checksum_worker, (name, g["blocks"], g["substreams"], g["T"]))
    want = (g["sum"], g["xor"], g["mant"])
    assert res[0] == want and res[1] == want


def _hwd_worker(rank, world, port, q, d):
    _init(rank, world, port)
    try:
        from paper_1805_01407_b200 import hwd

        rep = hwd.run_generator(d["name"], hwd.HwdConfig(**d["config"]), seed=d["seed"],
                                checkpoint_start=d["checkpoint_start"])
        q.put((rank, rep.to_dict()))
    finally:
        dist.destroy_process_group()


def test_hwd_two_ranks_on_gpu(G):
    key = "xoroshiro128plus/5/500000/byte_limit=32000000,k=6,mode=transitional,w=64"
    d = G("hwd")[key]
    want = {k: v for k, v in d.items() if k not in ("name", "seed", "checkpoint_start", "config", "ref_seconds")}
    res = _run(_hwd_worker, (d,))
    assert res[0] == want and res[1] == want

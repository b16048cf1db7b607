"""The NCCL collectives of the multi-GPU path, on the one GPU of this box:
a one-rank NCCL process group (one process per GPU, as bench.py launches
them) runs the config-5 checksum gather (collective_device -> CUDA tensors,
one all_gather) and the HWD counter all-reduce (uint64 counters on the
device).  With one rank the collectives are identities, so the results must
equal the reference's golden values; what this pins is that every tensor
handed to NCCL lives on the GPU and has a dtype NCCL reduces (VERDICT r1:
only gloo had ever run)."""

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


def _worker(port, q, c5, hwd_case):
    import sys

    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    try:
        # as bench.py initialises it (device_id binds the communicator eagerly)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        dist.barrier()
        import paper_1805_01407_b200 as P
        from paper_1805_01407_b200 import hwd
        from paper_1805_01407_b200.multigpu import _device_compute, collective_device, gather_checksums

        out = {"device": str(collective_device())}
        name, g = c5
        spec = P.get_spec(name)
        local = _device_compute(spec, 42, list(range(g["blocks"])), g["substreams"], g["T"])
        total, parts = gather_checksums(local, spec.kind.w)  # device=None: NCCL -> CUDA tensors
        out["c5"] = (hex(total.sum), hex(total.xor), hex(total.mant), len(parts))
        d = hwd_case
        rep = hwd.run_generator(d["name"], hwd.HwdConfig(**d["config"]), seed=d["seed"],
                                checkpoint_start=d["checkpoint_start"], group=dist.group.WORLD)
        out["hwd"] = rep.to_dict()

        # with one rank run_generator skips the all-reduce: drive the HWD
        # counter snapshot (device uint64 counters, NCCL all-reduce) directly
        class Counter:
            def totals(self):
                return (torch.tensor([(1 << 40) + i for i in range(5)], dtype=torch.uint64, device="cuda"),
                        torch.tensor([3 * i for i in range(5)], dtype=torch.uint64, device="cuda"))

        c, w = hwd._totals_async(Counter(), dist.group.WORLD)()
        out["hwd_allreduce"] = ([int(x) for x in c], [int(x) for x in w])
        q.put(out)
    except BaseException:
        import traceback

        q.put({"error": traceback.format_exc()})
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_nccl_one_rank_collectives(G):
    name = "xoshiro512starstar"
    g = G("checksums_small")[f"c5s/{name}"]
    key = "xoroshiro128plus/5/500000/byte_limit=32000000,k=6,mode=transitional,w=64"
    d = G("hwd")[key]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q, (name, g), d))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=120)
    assert "error" not in res, res.get("error")
    assert p.exitcode == 0
    assert res["device"] == "cuda:0"
    assert res["c5"] == (g["sum"], g["xor"], g["mant"], 1)
    want = {k: v for k, v in d.items() if k not in ("name", "seed", "checkpoint_start", "config", "ref_seconds")}
    assert res["hwd"] == want
    assert res["hwd_allreduce"] == ([(1 << 40) + i for i in range(5)], [3 * i for i in range(5)])

"""bench.py's launch contract on the host (no GPU): the N-GPU guard, the
reference arm's rank-0-only rule, and the JSON helpers the driver reads."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, **env):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(env)
    return subprocess.run([sys.executable, BENCH, *args], env=e, cwd=ROOT, capture_output=True, text=True,
                          timeout=300)


def test_refuses_a_world_size_other_than_gpus():
    r = _run(["--gpus", "2"], WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    assert r.returncode != 0
    assert "--gpus 2" in r.stderr and "WORLD_SIZE=1" in r.stderr
    assert r.stdout == ""


def test_reference_arm_runs_on_rank_zero_only():
    """Under torchrun the other ranks of the reference arm exit 0 without work or output."""
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"], WORLD_SIZE="2", RANK="1",
             LOCAL_RANK="1")
    assert r.returncode == 0, r.stderr
    assert r.stdout == ""


def test_config_and_committed_profile_inputs():
    sys.path.insert(0, ROOT)
    import bench

    cfg = bench.config(4)
    assert cfg["world_size"] == 4 and cfg["substreams_per_gpu"] == 1 << 20 and cfg["outputs_per_substream"] == 1024
    # roofline.traffic and the fused INT roofline come from committed ncu summaries
    assert bench.ncu_traffic("k_fill_xoshiro256starstar_u64_tma") > 8e9
    pipes = bench.fused_pipes()
    for mode in ("sum_xor", "exact", "exact_f64"):
        assert 10 < pipes[mode]["alu_sass_per_output"] < 30
    g = bench.golden_checksum("c2/xoshiro256starstar")
    assert g and g["sum"].startswith("0x") and g["xor"].startswith("0x")


@pytest.mark.parametrize("gpus", ["1"])
def test_one_gpu_needs_no_relaunch(gpus):
    sys.path.insert(0, ROOT)
    import bench

    class A:
        pass

    a = A()
    a.gpus = int(gpus)
    os.environ.pop("WORLD_SIZE", None)
    assert bench.relaunch_if_needed(a) is None
    json.dumps(bench.config(1))

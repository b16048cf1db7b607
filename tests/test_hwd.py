"""HWD consumer: host-side pieces (CPU) and the GPU counting path against
reports the reference's run_generator produced (tests/golden/hwd.json)."""

import math

import numpy as np
import pytest

from paper_1805_01407_b200 import hwd


def test_trit_mapping_and_ell():
    assert hwd.choose_ell(64) == 2 and hwd.choose_ell(32) == 1 and hwd.choose_ell(16) == 0
    assert hwd.trit_of(0, 64, 2) == 0
    assert hwd.trit_of((1 << 32) - 1, 64, 2) == 1
    assert hwd.trit_of((1 << 64) - 1, 64, 2) == 2
    assert hwd.trit_of((1 << 29) - 1, 64, 2) == 0 and hwd.trit_of((1 << 30) - 1, 64, 2) == 1
    assert hwd.trit_of((1 << 34) - 1, 64, 2) == 1 and hwd.trit_of((1 << 35) - 1, 64, 2) == 2
    assert hwd.central_probability(16, 0) == math.comb(16, 8) / 2 ** 16


def test_signature_and_format():
    assert hwd.signature_update(0, 2, 8) == 2 * 3 ** 7
    assert hwd.signature_update(3 ** 8 - 1, 0, 8) == 3 ** 7 - 1
    s = np.arange(0, 3 ** 12, dtype=np.uint64)
    assert np.array_equal((hwd.FIXED_POINT_RECIP * s) >> np.uint64(32), s // 3)
    assert hwd.format_signature(2 * 3 ** 7 + 1 * 3 ** 6, 8) == "00000012"
    assert hwd.format_signature(0, 4) == "0000"


def test_transform_orthogonal():
    for vec, want in [((1, 1, 1), (math.sqrt(3), 0, 0)), ((1, 0, -1), (0, math.sqrt(2), 0)),
                      ((1, -2, 1), (0, 0, -math.sqrt(6)))]:
        v = np.array(vec, dtype=float)
        hwd.transform(v)
        assert np.allclose(v, want, atol=1e-12)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(3 ** 5)
    n0 = np.linalg.norm(v)
    hwd.transform(v)
    assert abs(np.linalg.norm(v) - n0) < 1e-9
    with pytest.raises(ValueError):
        hwd.transform(np.zeros(10))


def test_evaluate_uniform_and_empty():
    cfg = hwd.HwdConfig(w=64, k=3)
    n = 27
    ck = hwd.evaluate_counts(np.zeros(n, np.uint64), np.zeros(n, np.uint64), cfg, 0)
    assert ck.p_value == 1.0
    cnt = np.full(n, 1000, np.uint64)
    ck = hwd.evaluate_counts(cnt, cnt * np.uint64(32), cfg, 27000)
    assert ck.p_value == 1.0


def test_config_validation():
    with pytest.raises(ValueError):
        hwd.HwdConfig(k=0)
    with pytest.raises(ValueError):
        hwd.HwdConfig(mode="weird")
    c = hwd.HwdConfig(w=32, k=6)
    assert c.ell == 1 and c.C == 4


def _cases(G):
    return G("hwd")


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(9))
def test_run_generator_matches_reference(G, idx):
    cases = sorted(G("hwd").items())
    if idx >= len(cases):
        pytest.skip("golden case not generated")
    key, d = cases[idx]
    if d["config"].get("batch_size") is not None:
        with pytest.warns(RuntimeWarning, match="batch_size is ignored"):
            cfg = hwd.HwdConfig(**d["config"])
    else:
        cfg = hwd.HwdConfig(**d["config"])
    rep = hwd.run_generator(d["name"], cfg, seed=d["seed"], checkpoint_start=d["checkpoint_start"]).to_dict()
    want = {k: v for k, v in d.items() if k not in ("name", "seed", "checkpoint_start", "config", "ref_seconds")}
    assert rep == want, key


@pytest.mark.gpu
def test_paper_row_xorshift128plus_transitional_detected():
    """test_hwd.py:286-296 of the reference (marked slow there: hours in numpy)."""
    with pytest.warns(RuntimeWarning):
        cfg = hwd.HwdConfig(w=64, k=8, byte_limit=int(2.4e10), batch_size=2_300_000, mode="transitional")
    rep = hwd.run_generator("xorshift128plus", cfg, seed=1, lanes=16384, lane_len=1024)
    assert rep.status == "failed"
    assert rep.bytes_processed <= 2.4e10
    assert rep.faulty_signature in ("00000012", "00000021")


@pytest.mark.gpu
def test_paper_row_xoshiro256starstar_passes():
    """test_hwd.py:298-304 of the reference."""
    with pytest.warns(RuntimeWarning):
        cfg = hwd.HwdConfig(w=64, k=8, byte_limit=int(1e10), batch_size=2_300_000)
    rep = hwd.run_generator("xoshiro256starstar", cfg, seed=1, lanes=16384, lane_len=1024)
    assert rep.status == "passed"
    assert rep.p_value > 1e-20

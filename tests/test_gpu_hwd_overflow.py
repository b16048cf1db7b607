"""K6 exactness when the packed 13/19-bit shared counters overflow: a launch
with far too many values per CTA for 9 signatures (k = 2) must fall back to
the in-kernel 64-bit recount and give the same counts as safe launches."""

import numpy as np
import pytest

from paper_1805_01407_b200 import hwd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,split", [("standard", False), ("transitional", True)])
def test_overflowing_ctas_recount_exactly(mode, split):
    w = 32 if split else 64
    cfg = hwd.HwdConfig(w=w, k=2, mode=mode, split=split)
    c0, c1 = 2, 2 + 256 * 40_000
    W = cfg.k + (1 if mode == "transitional" else 0)
    if split:
        W += (c0 - W) & 1
    safe = hwd._GpuCounter(hwd.get_spec("xoshiro256plus"), 5, cfg)
    safe.count(c0, c1)                                   # host-sized segments: no overflow
    big = hwd._GpuCounter(hwd.get_spec("xoshiro256plus"), 5, cfg)
    big._launch(c0, c1, 40_000, 256, W)                  # one CTA, 1e7 values over 9 cells: overflows
    a_cnt, a_sum = safe.snapshot()
    b_cnt, b_sum = big.snapshot()
    assert int(big.overflow.cpu().numpy()[0]) >= 1
    assert int(safe.overflow.cpu().numpy()[0]) == 0
    np.testing.assert_array_equal(a_cnt, b_cnt)
    np.testing.assert_array_equal(a_sum, b_sum)
    assert int(a_cnt.sum()) == c1 - c0


@pytest.mark.parametrize("k,mode,split", [(10, "standard", False), (11, "transitional", False),
                                          (10, "standard", True), (12, "standard", False)])  # k=12: global path
def test_sliced_cells_equal_global_atomics_and_oracle(k, mode, split):
    """k >= 10: 3^k cells split over CTA slices in shared memory (each slice
    regenerates its segments) give exactly the counts of 64-bit global atomics
    (SLP_HWD_SLICES=0) and of the CPU oracle."""
    import os

    from oracle import oracle as O

    w = 32 if split else 64
    cfg = hwd.HwdConfig(w=w, k=k, mode=mode, split=split)
    spec = hwd.get_spec("xoroshiro128plus")
    c0, c1 = k, 300_000
    res = {}
    for flag in ("1", "0"):
        old = os.environ.get("SLP_HWD_SLICES")
        os.environ["SLP_HWD_SLICES"] = flag
        try:
            ctr = hwd._GpuCounter(spec, 3, cfg)
            ctr.count(c0, c1)
            res[flag] = ctr.snapshot()
        finally:
            if old is None:
                del os.environ["SLP_HWD_SLICES"]
            else:
                os.environ["SLP_HWD_SLICES"] = old
    np.testing.assert_array_equal(res["1"][0], res["0"][0])
    np.testing.assert_array_equal(res["1"][1], res["0"][1])
    assert int(res["1"][0].sum()) == c1 - c0
    vals = O.hwd_test_values("xoroshiro128plus", 3, c1, split, mode == "transitional", w)
    want_c, want_s = O.hwd_counts(vals, c0, c1, k, w, cfg.ell)
    np.testing.assert_array_equal(res["1"][0], want_c)
    np.testing.assert_array_equal(res["1"][1], want_s)

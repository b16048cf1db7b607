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

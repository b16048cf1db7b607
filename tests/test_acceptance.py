"""The reference's hot-path acceptance criteria (SURVEY.md section 4,
test_acceptance.py:34-46 and :283-330), restated against the oracle:

* criterion 1: every registry generator, seed 1, the first 10^4 outputs of
  its stream -- here produced by the GPU bulk path (output_stream, kernels
  K1 + K2) and by the host scalar Generator;
* criterion 11: the default jump and long jump for 10 seeds per engine
  (host jump in C++ vs the oracle's polynomial jump)."""

import numpy as np
import pytest

import paper_1805_01407_b200 as P
from oracle import oracle as O

NAMES = P.registry_names()  # the 25 production generators


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_criterion1_bulk_stream(name):
    spec = P.get_spec(name)
    want = O.laned_stream(name, 1, 10_000, 64, 256)
    got = np.concatenate(list(P.output_stream(spec, seed=1, total_values=10_000, lanes=64, lane_len=256)))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("name", NAMES)
def test_criterion1_scalar_stream(name):
    spec = P.get_spec(name)
    g = P.Generator.from_seed(spec, 1)
    got = np.array([g.next() for _ in range(2_000)], dtype=np.uint64)
    want = O.laned_stream(name, 1, 2_000, 1, 2_000)
    np.testing.assert_array_equal(got, want)


ENGINES = ["xoroshiro128plus", "xoshiro256plus", "xoshiro512plus", "xoroshiro1024plus", "xoroshiro64star",
           "xoshiro128plus", "xoroshiro128plusplus"]


@pytest.mark.parametrize("name", ENGINES)
def test_criterion11_default_jumps_ten_seeds(name):
    spec = P.get_spec(name)
    jump, long_jump = P.default_jumps(spec)
    n = spec.kind.n
    pj = O.jump_poly(name, 1 << (n // 2))
    plj = O.jump_poly(name, 1 << (3 * n // 4))
    assert jump.poly.bits == pj and long_jump.poly.bits == plj
    for seed in range(10):
        g = P.Generator.from_seed(spec, seed)
        flat = list(g.flat_words())
        g.jump(jump)
        assert list(g.flat_words()) == O.jump(name, flat, pj), (name, seed)
        g2 = P.Generator.from_seed(spec, seed)
        g2.jump(long_jump)
        assert list(g2.flat_words()) == O.jump(name, flat, plj), (name, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("name,lanes,lane_len", [("xoshiro256starstar", 512, 8192), ("xoroshiro128plus", 64, 1 << 14),
                                                 ("xoshiro128starstar", 256, 4096)])
def test_laned_stream_through_the_segment_split(name, lanes, lane_len):
    """LanedStream geometries below one wave of lanes: the C ABI splits every
    lane into jumped segments; two superbatches (super-jump between them)
    must still equal the reference's laned stream."""
    from paper_1805_01407_b200 import device as D

    spec = P.get_spec(name)
    assert D._split_factor(spec, lanes, lane_len, "stream", lane_len) > 1
    total = 2 * lanes * lane_len - 777
    want = O.laned_stream(name, 5, total, lanes, lane_len)
    got = np.concatenate(list(P.output_stream(spec, seed=5, total_values=total, lanes=lanes, lane_len=lane_len)))
    np.testing.assert_array_equal(got, want)

"""K1 lane split (k_jump, JumpParams::parts): a jump of an 8- or 16-word
engine shared by 2, 4 or 8 adjacent lanes must give the states of the
one-lane kernel and of the host jumps (Generator.jump, generators.py:315-334),
for every launch kind: per-lane polynomials (direct launch), uniform rounds,
slp_jump_states and the segment split of a single stream."""
import os

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

WIDE = ["xoroshiro1024plusplus", "xoroshiro1024star", "xoshiro512starstar", "xoshiro512plus"]


class forced:
    def __init__(self, **env):
        self.env = env

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.env}
        os.environ.update({k: str(v) for k, v in self.env.items()})

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def states(spec, n, blocks=1):
    sub = D.Substreams.from_seed(spec, 42, n, blocks=blocks)
    torch.cuda.synchronize()
    return sub.states.cpu().numpy().astype(np.uint64)


@pytest.mark.parametrize("name", WIDE)
@pytest.mark.parametrize("parts", [2, 4, 8])
def test_init_states_equal_one_lane_kernel(name, parts):
    spec = P.get_spec(name)
    for n, blocks in ((1, 1), (37, 3), (1000, 1), (5001, 2)):  # direct launch only ... direct + rounds
        with forced(SLP_JUMP_PARTS=1, SLP_INIT_TABLES=0):
            want = states(spec, n, blocks)
        with forced(SLP_JUMP_PARTS=parts, SLP_INIT_TABLES=0):
            got = states(spec, n, blocks)
        np.testing.assert_array_equal(got, want)
    nb = spec.kind.n
    for i in (0, 1, 4095, 4096, 5000):
        g = P.Generator.from_seed(spec, 42)
        if i:
            g.jump(P.compute_jump_poly(spec, i << (nb // 2)))
        assert list(g.flat_words()) == [int(v) for v in got[:, i]], i


@pytest.mark.parametrize("name", ["xoroshiro1024plusplus", "xoshiro512starstar"])
@pytest.mark.parametrize("parts", [2, 8])
def test_jump_states_and_single_stream_split(name, parts):
    spec = P.get_spec(name)
    jp = P.compute_jump_poly(spec, 987654321)
    short = P.compute_jump_poly(spec, 5)  # low degree: most lanes of a split jump have no coefficients
    with forced(SLP_JUMP_PARTS=parts):
        sub = D.Substreams.from_seed(spec, 7, 300)
        S0 = sub.states_numpy().astype(np.uint64)
        sub.jump(jp)
        S1 = sub.states_numpy().astype(np.uint64)
        sub.jump(short)
        S2 = sub.states_numpy().astype(np.uint64)
        one = D.Substreams.from_states(spec, S0[:, :1].copy())
        assert D._split_factor(spec, 1, 1 << 16, "stream", 1 << 16) > 1
        out = one.fill(1 << 16).cpu().numpy()
        end = one.states_numpy().astype(np.uint64)
    for i in (0, 1, 299):
        g = P.Generator.from_seed(spec, 0)
        g.set_flat_words([int(v) for v in S0[:, i]])  # flat order (the constructor takes ring storage order)
        g.jump(jp)
        assert list(g.flat_words()) == [int(v) for v in S1[:, i]]
        for _ in range(5):
            g.next()
        assert list(g.flat_words()) == [int(v) for v in S2[:, i]]
    want, want_end = O.vec_outputs(name, S0[:, :1], 1 << 16)
    np.testing.assert_array_equal(out, want)
    np.testing.assert_array_equal(end, want_end)


def test_custom_wide_engine_split():
    """Run-time parameter instance of an 8-word engine (GenR) through the split."""
    spec = P.custom_spec("xoshiro", 8, 64, 13, 31, scrambler=P.ScramblerSpec("plus", word_i=0, word_j=2),
                         name="xoshiro512-custom-13-31")
    with forced(SLP_JUMP_PARTS=1):
        want = states(spec, 700)
    for parts in (2, 4, 8):
        with forced(SLP_JUMP_PARTS=parts):
            np.testing.assert_array_equal(states(spec, 700), want)

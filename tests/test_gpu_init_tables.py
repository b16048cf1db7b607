"""K1t (table-driven uniform jump, four Russians) against K1 (polynomial
jump) and against host jumps: substream initialisation must give the same
states whichever kernel runs the radix rounds (SLP_INIT_TABLES=0 forces K1)."""
import os

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D

pytestmark = pytest.mark.gpu

# one generator per engine (jump tables belong to the engine)
ENGINES = ["xoroshiro128plus", "xoshiro256starstar", "xoshiro512plusplus", "xoroshiro1024starstar",
           "xoroshiro64star", "xoshiro128plusplus", "xorshift128plus"]


def _init(spec, n, blocks, tables):
    old = os.environ.get("SLP_INIT_TABLES")
    os.environ["SLP_INIT_TABLES"] = "1" if tables else "0"
    try:
        sub = D.Substreams.from_seed(spec, 42, n, blocks=blocks)
        torch.cuda.synchronize()
        return sub.states.cpu().numpy().astype(np.uint64)
    finally:
        if old is None:
            del os.environ["SLP_INIT_TABLES"]
        else:
            os.environ["SLP_INIT_TABLES"] = old


@pytest.mark.parametrize("name", ENGINES)
def test_tables_equal_polynomial_rounds(name):
    spec = P.get_spec(name)
    n, blocks = 40000, 2  # the last radix round (>= 16384 states) runs on K1t
    a = _init(spec, n, blocks, True)
    b = _init(spec, n, blocks, False)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro1024starstar", "xoshiro128plusplus"])
def test_tables_match_host_jumps(name):
    spec = P.get_spec(name)
    n = 40000
    S = _init(spec, n, 2, True)
    nb = spec.kind.n
    jump, long_jump = P.default_jumps(spec)
    for b in (0, 1):
        for i in (0, 1, 8191, 8192, 20000, n - 1):
            g = P.Generator.from_seed(spec, 42)
            if b:
                g.jump(long_jump)
            if i:
                g.jump(P.compute_jump_poly(spec, i << (nb // 2)))
            assert list(g.flat_words()) == [int(v) for v in S[:, b * n + i]], (b, i)


@pytest.mark.parametrize("name", ENGINES)
def test_jump_states_tables_equal_polynomial(name):
    """slp_jump_states on >= 65536 states uses K1t with a cached table (in
    place for n <= 256, out of place above); equal to K1."""
    spec = P.get_spec(name)
    jp = P.compute_jump_poly(spec, 987654321987654321)
    base = D.Substreams.from_seed(spec, 5, 70000)
    res = {}
    for flag in ("1", "0"):
        old = os.environ.get("SLP_INIT_TABLES")
        os.environ["SLP_INIT_TABLES"] = flag
        try:
            sub = D.Substreams(spec, base.states.clone(), base.count)
            sub.jump(jp)
            sub.jump(jp)  # second call: cached table
            torch.cuda.synchronize()
            res[flag] = sub.states.cpu().numpy()
        finally:
            if old is None:
                del os.environ["SLP_INIT_TABLES"]
            else:
                os.environ["SLP_INIT_TABLES"] = old
    assert np.array_equal(res["1"], res["0"])
    # spot check against the host jump
    S0 = base.states.cpu().numpy().astype(np.uint64)
    for i in (0, 12345, 69999):
        g = P.Generator(spec, [int(v) for v in S0[:, i]], ptr=spec.kind.k - 1)
        g.jump(jp)
        g.jump(jp)
        assert list(g.flat_words()) == [int(v) for v in res["1"][:, i].astype(np.uint64)]

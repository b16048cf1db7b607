"""custom_spec engines (generators.py:127-135), host side (no GPU).

The oracle's restatement is pinned against the reference's own outputs for
custom engines (tests/golden/custom.json, made by make_golden_custom.py);
the package's host algebra (char / jump polynomials, scalar Generator, host
jump) and the C ABI registration (slp_register_generator) are checked
against the same fixtures."""

import ctypes

import numpy as np
import pytest

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import _native
from paper_1805_01407_b200.generators import native_id
from oracle import oracle as O

NAMES = list(__import__("json").load(open(__import__("os").path.join(
    __import__("os").path.dirname(__file__), "golden", "custom.json"))))


def spec_of(d, name):
    sc = P.ScramblerSpec(**d["scrambler"])
    return P.custom_spec(d["family"], d["k"], d["w"], d["a"], d["b"], d["c"], scrambler=sc, name=name)


def hexs(vs):
    return [hex(int(v)) for v in vs]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_pinned_to_reference(G, name):
    d = G("custom")[name]
    n = d["k"] * d["w"]
    flat = O.seed_flat(name, 42)
    outs, _ = O.outputs(name, flat, 100)
    assert hexs(outs) == d["first_outputs_seed42"]
    assert O.jump_poly(name, 1 << (n // 2)) == int(d["jump_poly"], 16)
    S = O.lane_states(name, flat, 40, 1 << (n // 2))
    assert [hexs(S[:, i]) for i in range(40)] == d["substreams"]
    S2 = S.copy()
    for _ in range(64):
        S2 = O.vec_step(name, S2)
    assert [hexs(S2[:, i]) for i in range(40)] == d["substreams_after_64"]
    assert hexs(O.laned_stream(name, 42, 3000, 5, 512)) == d["laned_3000"]


@pytest.mark.parametrize("name", NAMES)
def test_host_algebra_and_scalar(G, name):
    d = G("custom")[name]
    spec = spec_of(d, name)
    n = spec.kind.n
    assert P.engine_char_poly(spec).bits == int(d["char_poly"], 16)
    jp = P.compute_jump_poly(spec, 1 << (n // 2))
    assert jp.poly.bits == int(d["jump_poly"], 16)
    g = P.Generator.from_seed(spec, 42)
    assert [hex(g.next()) for _ in range(100)] == d["first_outputs_seed42"]
    # host jump through the registered custom id == substream 1 of the laned set-up
    g = P.Generator.from_seed(spec, 42)
    g.jump(jp)
    assert hexs(g.flat_words()) == d["substreams"][1]


def test_registration_ids_and_info(G):
    d = G("custom")["xoroshiro128plus-2016"]
    spec = spec_of(d, "xoroshiro128plus-2016")
    gid = native_id(spec)
    assert gid >= 1024
    assert native_id(spec) == gid  # idempotent
    info = _native.GenInfo()
    _native.check(_native.lib().slp_generator_info(gid, ctypes.byref(info)), "info")
    assert (info.family, info.k, info.w, info.a, info.b, info.c) == (0, 2, 64, 55, 14, 36)
    assert (info.scrambler, info.word_i, info.word_j) == (1, 0, 1)
    assert info.name.decode() == "xoroshiro128plus-2016"
    # a custom spec with registry parameters maps to the registry id
    reg = P.get_spec("xoshiro256starstar")
    same = P.custom_spec("xoshiro", 4, 64, 17, 45, scrambler=reg.scrambler, name="mine")
    assert native_id(same) == 8


def test_registration_validation():
    L = _native.lib()

    def reg(**kw):
        info = _native.GenInfo()
        base = dict(family=1, k=4, w=64, a=17, b=45, c=0, scrambler=4, word_i=1, word_j=-1, R=7, S=5, T=9)
        base.update(kw)
        for k, v in base.items():
            setattr(info, k, v)
        info.name = b"t"
        return L.slp_register_generator(ctypes.byref(info))

    assert reg() == 8  # == xoshiro256starstar
    assert reg(S=4) == _native.SLP_ERR_INVALID     # even multiplier (scramblers.py:76-77)
    assert reg(R=64) == _native.SLP_ERR_INVALID    # rotation out of range
    assert reg(T=2) == _native.SLP_ERR_INVALID
    assert reg(word_i=4) == _native.SLP_ERR_INVALID
    assert reg(scrambler=1, word_j=9) == _native.SLP_ERR_INVALID
    assert reg(k=5) == _native.SLP_ERR_INVALID     # xoshiro only k in {4, 8}
    assert reg(a=0) == _native.SLP_ERR_INVALID     # engines.py:89-97
    assert reg(family=0, c=0) == _native.SLP_ERR_INVALID
    assert L.slp_register_generator(None) == _native.SLP_ERR_INVALID


def test_engines_exports_vecstepper():
    from paper_1805_01407_b200 import engines

    assert "VecStepper" in engines.__all__
    from paper_1805_01407_b200.device import VecStepper

    assert engines.VecStepper is VecStepper
    st = engines.VecStepper(P.EngineKind("xoroshiro", 2, 64), P.EngineParams(55, 14, 36))
    assert st.spec.kind.k == 2
    with pytest.raises(ValueError):
        engines.VecStepper(P.EngineKind("xoroshiro", 2, 16), P.EngineParams(3, 5, 7))
    assert isinstance(np.uint64(0), np.uint64)

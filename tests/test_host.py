"""Host side of the drop-in (no GPU): registry, seeding, scalar Generator,
GF(2) jump machinery from the native host library, error behaviour.
Mirrors the reference's own tests (test_generators.py, test_engines.py,
test_scramblers.py) against the golden vectors."""

import ctypes
import random

import pytest

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import _native
from paper_1805_01407_b200.engines import EngineKind, EngineParams, rotl, step

ALL = P.registry_names(include_analysis=True)


def hexs(vals):
    return [hex(int(v)) for v in vals]


def test_registry_names():
    assert len(P.REGISTRY) == 25 and len(P.ANALYSIS_REGISTRY) == 2
    assert P.get_spec("xoroshiro128plusplus").params == EngineParams(49, 21, 28)
    assert P.get_spec("xoshiro512plus").scrambler.word_j == 2
    with pytest.raises(KeyError):
        P.get_spec("mt19937")


def test_registry_matches_native_table():
    """The Python table and csrc/slp_registry.h describe the same generators, in id order."""
    L = _native.lib()
    assert L.slp_num_generators() == 27
    kinds = ["none", "plus", "star", "plusplus", "starstar"]
    fams = ["xoroshiro", "xoshiro", "xorshift"]
    for i, name in enumerate(ALL):
        info = _native.GenInfo()
        assert L.slp_generator_info(i, ctypes.byref(info)) == 0
        assert L.slp_generator_id(name.encode()) == i
        s = P.get_spec(name)
        assert info.name.decode() == name
        assert (fams[info.family], info.k, info.w) == (s.kind.family, s.kind.k, s.kind.w)
        assert (info.a, info.b) == (s.params.a, s.params.b)
        assert info.c == (s.params.c or 0)
        sc = s.scrambler
        assert kinds[info.scrambler] == sc.kind and info.word_i == sc.word_i
        assert info.word_j == (-1 if sc.word_j is None else sc.word_j)
        assert info.S == (sc.S or 0) and info.R == (sc.R or 0) and info.T == (sc.T or 0)
    assert L.slp_generator_id(b"nope") == _native.SLP_ERR_UNKNOWN_GENERATOR


def test_splitmix_and_seeding(G):
    mix = P.splitmix64(0)
    assert next(mix) == 0xE220A8397B1DCDAF and next(mix) == 0x6E789E6AA1B965F4
    for name in ALL:
        for seed, want in G("generators")[name]["seed_states"].items():
            assert hexs(P.seed_state(P.get_spec(name), int(seed))) == want


@pytest.mark.parametrize("name", ALL)
def test_scalar_generator(G, name):
    d = G("generators")[name]
    spec = P.get_spec(name)
    for seed in (42, 7):
        g = P.Generator.from_seed(spec, seed)
        assert hexs(g.next() for _ in range(100)) == d[f"first_outputs_seed{seed}"]
        assert hexs(g.flat_words()) == d[f"state_after_100_seed{seed}"]
    if spec.kind.w == 64:
        g = P.Generator.from_seed(spec, 42)
        assert [float.hex(g.next_double()) for _ in range(16)] == d["first_doubles_seed42"]
    else:
        with pytest.raises(ValueError):
            P.Generator.from_seed(spec, 1).next_double()


def test_char_and_jump_polys(G):
    for key, e in G("engines").items():
        spec = P.get_spec(e["generators"][0])
        assert hex(P.engine_char_poly(spec).bits) == e["char_poly"]
        j, lj = P.default_jumps(spec)
        assert hex(j.poly.bits) == e["jump_poly"] and hex(lj.poly.bits) == e["long_jump_poly"]
        assert j.step_count == 1 << (spec.kind.n // 2) and lj.step_count == 1 << (3 * spec.kind.n // 4)
        for steps, field in ((1024, "x_pow_1024"), (4096, "x_pow_4096"), (12345, "x_pow_12345")):
            assert hex(P.compute_jump_poly(spec, steps).poly.bits) == e[field]


@pytest.mark.parametrize("name", ALL)
def test_jump_states(G, name):
    d = G("generators")[name]
    spec = P.get_spec(name)
    j, lj = P.default_jumps(spec)
    g = P.Generator.from_seed(spec, 42).jump(j)
    assert hexs(g.flat_words()) == d["jump_state_seed42"]
    assert hexs(g.next() for _ in range(32)) == d["jump_outputs_seed42"][:32]
    g = P.Generator.from_seed(spec, 42).jump(lj)
    assert hexs(g.flat_words()) == d["long_jump_state_seed42"]


def test_substream_states_sparse(G):
    for name, d in G("substreams").items():
        spec = P.get_spec(name)
        J = 1 << (spec.kind.n // 2)
        for idx, want in d["sparse_states"].items():
            g = P.Generator.from_seed(spec, d["seed"]).jump(P.compute_jump_poly(spec, int(idx) * J))
            assert hexs(g.flat_words()) == want


def test_jump_trivia_and_errors():
    spec = P.get_spec("xoroshiro128")
    assert P.compute_jump_poly(spec, 0).poly == P.GF2Poly(1)
    assert P.compute_jump_poly(spec, 1).poly == P.GF2Poly(2)
    with pytest.raises(ValueError):
        P.compute_jump_poly(spec, -1)
    g = P.Generator.from_seed(P.get_spec("xoshiro256plus"), 1)
    with pytest.raises(ValueError):
        g.jump(P.compute_jump_poly(spec, 5))
    spec2 = P.get_spec("xoshiro256plus")
    g1 = P.Generator.from_seed(spec2, 9)
    g2 = g1.clone()
    g1.jump(P.compute_jump_poly(spec2, 1))
    g2.next()
    assert g1.flat_words() == g2.flat_words()


def test_toy_jump_vs_stepping():
    """test_generators.py:153-165 on a custom 10-bit engine (not primitive-checked)."""
    spec = P.custom_spec("xoroshiro", 2, 5, 1, 3, 1, P.ScramblerSpec("plus", 0, 1))
    rng = random.Random(12)
    for _ in range(25):
        J, T = rng.randrange(1 << 10), rng.randrange(100)
        g1 = P.Generator(spec, [rng.randrange(1, 32), rng.randrange(32)])
        g2 = g1.clone()
        g1.jump(P.compute_jump_poly(spec, J))
        for _ in range(T):
            g1.next()
        for _ in range(J + T):
            g2.next()
        assert g1.flat_words() == g2.flat_words()


def test_generator_validation():
    spec = P.get_spec("xoshiro256plus")
    with pytest.raises(ValueError):
        P.Generator(spec, [0, 0, 0, 0])
    with pytest.raises(ValueError):
        P.Generator(spec, [1, 2, 3])
    with pytest.raises(ValueError):
        P.Generator(spec, [1 << 64, 0, 0, 0])
    with pytest.raises(ValueError):
        P.Generator(P.get_spec("xoroshiro1024"), [1] * 16, ptr=16)
    ring_bad = P.custom_spec("xoroshiro", 16, 64, 25, 27, 36, P.ScramblerSpec("plus", 0, 5))
    with pytest.raises(ValueError):
        P.Generator(ring_bad, [1] * 16)
    with pytest.raises(ValueError):
        EngineKind("xoshiro", 3, 64)
    with pytest.raises(ValueError):
        P.ScramblerSpec("star", 0, S=4).validate(2, 64)


def test_engine_step_traces():
    assert step(EngineKind("xoroshiro", 2, 64), EngineParams(24, 16, 37), (1, 0)) == (0x1010001, 0x2000000000)
    assert step(EngineKind("xoshiro", 4, 64), EngineParams(17, 45), (1, 0, 0, 0)) == (1, 1, 1, 0)
    assert rotl(1 << 63, 1, 64) == 1
    with pytest.raises(ValueError):
        rotl(1, 64, 64)


def test_kats():
    assert P.Generator(P.get_spec("xoroshiro128plus"), [1, 2]).next() == 3
    assert P.Generator(P.get_spec("xoshiro256starstar"), [0, 1, 0, 0]).next() == 5760
    spec = P.get_spec("xoroshiro128plus")
    assert P.Generator(spec, [1, (1 << 64) - 1]).next_double() == 0.0
    assert P.Generator(spec, [1 << 63, 0]).next_double() == 0.5
    assert P.Generator(spec, [(1 << 64) - 1, 0]).next_double() == (2 ** 53 - 1) / 2 ** 53


def test_ring_pointer_forms_agree():
    """test_engines.py:90-103: pointer storage vs flat step."""
    spec = P.get_spec("xoroshiro1024starstar")
    g = P.Generator.from_seed(spec, 99)
    words = tuple(g.flat_words())
    outs = [g.next() for _ in range(200)]
    ref = []
    for _ in range(200):
        ref.append(spec.scrambler.apply(words, 64))
        words = step(spec.kind, spec.params, words)
    assert outs == ref


@pytest.mark.parametrize("name,n,stride", [
    ("xoroshiro1024plusplus", 100, 1 << 512),      # small plan: 128 direct polynomials
    ("xoroshiro1024plusplus", 5000, 1 << 512),     # big plan: 4096 direct (threaded build), then rounds
    ("xoshiro512starstar", 40000, (1 << 256) + 12345),
    ("xoshiro256starstar", 3000, 1 << 128),
    ("xoroshiro64starstar", 3000, 977),
])
def test_init_plan_polynomials(name, n, stride):
    """The substream-initialisation plan (slp_init_substreams) holds x^(i*stride)
    mod P for i < direct, then the radix-8 round polynomials x^(c*m*stride):
    checked against compute_jump_poly (generators.py:397-402), including the
    block boundaries of the threaded build of large plans."""
    spec = P.get_spec(name)
    gid = _native.lib().slp_generator_id(name.encode())
    sw, sn = _native.int_to_words(stride)
    pw = (spec.kind.n + 63) // 64
    buf = (ctypes.c_uint64 * pw)()

    def plan_poly(i):
        cnt = _native.lib().slp_init_plan_poly(gid, sw, sn, n, i, buf, pw)
        assert cnt > 0
        return cnt, _native.words_to_int(buf)

    count, p0 = plan_poly(0)
    assert p0 == 1
    small = {256: 1024, 512: 256, 1024: 128}.get(spec.kind.n, 1024)
    direct = small if n <= small or spec.kind.n <= 256 else 4096
    direct = min(direct, count)
    rng = random.Random(n)
    idx = {1, 2, direct - 1, direct // 2, direct // 2 - 1, direct // 2 + 1} | {direct * j // 16 for j in range(1, 16)} \
        | {direct * j // 16 - 1 for j in range(1, 16)} | {direct * j // 8 + 1 for j in range(1, 8)} \
        | {rng.randrange(direct) for _ in range(8)}
    for i in sorted(i for i in idx if 0 <= i < direct):
        assert plan_poly(i)[1] == P.compute_jump_poly(spec, i * stride).poly.bits, (name, i)
    # the rounds (plans are built for direct * 8^r >= n): 7 polynomials x^(c * m * stride) each
    m, at = direct, direct
    while m < n:
        for c in range(1, 8):
            assert plan_poly(at)[1] == P.compute_jump_poly(spec, c * m * stride).poly.bits, (name, m, c)
            at += 1
        m *= 8
    assert at == count
    assert _native.lib().slp_init_plan_poly(gid, sw, sn, n, count + 5, None, 0) == count  # out of range: count only


def test_native_host_jump_errors():
    L = _native.lib()
    st = (ctypes.c_uint64 * 4)(0, 0, 0, 0)
    poly = (ctypes.c_uint64 * 4)(2, 0, 0, 0)
    assert L.slp_host_jump(6, poly, 4, st) == _native.SLP_ERR_ZERO_STATE
    zero = (ctypes.c_uint64 * 4)(0, 0, 0, 0)
    st2 = (ctypes.c_uint64 * 4)(1, 0, 0, 0)
    assert L.slp_host_jump(6, zero, 4, st2) == _native.SLP_ERR_ZERO_STATE
    assert L.slp_host_jump(99, poly, 4, st2) == _native.SLP_ERR_UNKNOWN_GENERATOR
    buf = (ctypes.c_uint64 * 2)()
    assert L.slp_char_poly(8, buf, 2) == _native.SLP_ERR_BUFFER
    with pytest.raises(ValueError):
        _native.check(_native.SLP_ERR_INVALID, "x")
    with pytest.raises(KeyError):
        _native.check(_native.SLP_ERR_UNKNOWN_GENERATOR, "x")
    with pytest.raises(_native.Gf2Error):
        _native.check(_native.SLP_ERR_ALGEBRA, "x")


def test_device_api_requires_gpu_when_absent():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1805_01407_b200 import device as D

    with pytest.raises(RuntimeError):
        D.Substreams.from_seed(P.get_spec("xoshiro256starstar"), 42, 4)
    with pytest.raises(RuntimeError):
        next(iter(P.output_stream(P.get_spec("xoshiro256starstar"), seed=1, total_values=10)))

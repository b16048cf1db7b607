"""Seeded random sweep over the fill parameter space against the oracle:
generator, substream count, row length (short rows, whole tiles, tails),
layout, output kind, row pitch (padding) and an element offset of the output
(alignment: TMA, staged and direct paths), with and without state
write-back.  Every case is bit-exact or the test fails with its parameters."""

import os

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ALL = P.registry_names(include_analysis=True)


def _case(rng):
    name = ALL[rng.integers(len(ALL))]
    n = int(rng.choice([1, 31, 32, 33, 100, 257, 1000, 5000]))
    T = int(rng.choice([1, 2, 15, 16, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 255, 256, 300, 511, 512, 513,
                        1000, 1024, 1151]))
    layout = str(rng.choice(["stream", "position"]))
    pad = int(rng.choice([0, 0, 0, 1, 3, 16]))
    off = int(rng.choice([0, 0, 0, 1, 2]))
    advance = bool(rng.integers(2))
    return name, n, T, layout, pad, off, advance


@pytest.mark.parametrize("seed", range(int(os.environ.get("SLP_FUZZ_SEEDS", "12"))))
def test_fill_fuzz(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(12):
        name, n, T, layout, pad, off, advance = _case(rng)
        spec = P.get_spec(name)
        w = spec.kind.w
        kinds = ["native", "f64"] if w == 64 else ["native", "u64", "f32"]
        kind = kinds[rng.integers(len(kinds))]
        flat = rng.integers(0, 1 << 63, size=(spec.kind.k, n), dtype=np.uint64) | np.uint64(1)
        if w == 32:
            flat &= np.uint64(0xFFFFFFFF)
        want, want_S = O.vec_outputs(name, flat, T)
        want = want.astype(np.uint64 if w == 64 else np.uint32)
        if kind == "u64":
            want = want.astype(np.uint64)
        elif kind == "f64":
            want = O.to_f64(want)
        elif kind == "f32":
            want = O.to_f32(want)
        if layout == "position":
            want = want.T.copy()
        rows, cols = want.shape
        dt = {np.dtype(np.uint64): torch.uint64, np.dtype(np.uint32): torch.uint32,
              np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}[want.dtype]
        big = torch.zeros((rows, cols + pad + off), dtype=dt, device="cuda")
        out = big[:, off:off + cols]
        sub = D.Substreams.from_states(spec, flat)
        D.fill(spec, sub.states, T, out=out, kind=kind, layout=layout, advance=advance)
        got = out.cpu().numpy()
        msg = f"{name} n={n} T={T} {layout} {kind} pad={pad} off={off} advance={advance}"
        np.testing.assert_array_equal(got.view(np.uint8), want.view(np.uint8), err_msg=msg)
        states = sub.states.cpu().numpy().astype(np.uint64)
        np.testing.assert_array_equal(states, want_S if advance else flat, err_msg=msg)
        if pad or off:  # nothing outside the output view is touched
            rest = big.cpu().numpy().view(np.uint8).reshape(rows, -1)
            es = big.element_size()
            assert not rest[:, : off * es].any() and not rest[:, (off + cols) * es:].any(), msg


@pytest.mark.parametrize("seed", range(int(os.environ.get("SLP_FUZZ_SEEDS", "12"))))
def test_checksum_fuzz(seed):
    """Fused consumer (K4) and store + checksum (K2 CSUM) on random shapes."""
    rng = np.random.default_rng(5000 + seed)
    for _ in range(8):
        name = ALL[rng.integers(len(ALL))]
        spec = P.get_spec(name)
        w = spec.kind.w
        n = int(rng.choice([1, 32, 45, 300, 3000]))
        T = int(rng.choice([1, 16, 17, 100, 128, 129, 512, 1000, 1024]))
        flat = rng.integers(0, 1 << 63, size=(spec.kind.k, n), dtype=np.uint64) | np.uint64(1)
        if w == 32:
            flat &= np.uint64(0xFFFFFFFF)
        want, want_S = O.vec_outputs(name, flat, T)
        oc = O.checksum(want, w)
        msg = f"{name} n={n} T={T}"
        c = D.Substreams.from_states(spec, flat).checksum(T, exact=True, f64=bool(rng.integers(2)))
        assert (c.sum, c.xor, c.mant) == (oc["sum"], oc["xor"], oc["mant"]), msg
        sub = D.Substreams.from_states(spec, flat)
        kind = "native" if rng.integers(2) else ("f64" if w == 64 else "f32")
        out, c2 = D.fill_checksum(spec, sub.states, T, kind=kind)
        assert (c2.sum, c2.xor, c2.mant) == (oc["sum"], oc["xor"], oc["mant"]), msg + " " + kind
        np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S, err_msg=msg)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SLP_FUZZ_SEEDS", "12")) // 3 + 1))
def test_init_fuzz(seed):
    """Substream set-up (K1 + K1t) with random strides, block strides and
    counts, sampled against host jumps (Generator.jump, generators.py:315-334)."""
    rng = np.random.default_rng(9000 + seed)
    for _ in range(3):
        name = ALL[rng.integers(len(ALL))]
        spec = P.get_spec(name)
        nb = spec.kind.n
        n = int(rng.choice([1, 7, 1000, 20000, 70000]))
        blocks = int(rng.choice([1, 2, 3]))
        stride = int(rng.integers(1, 1 << 62)) << int(rng.integers(0, nb // 2))
        bstride = int(rng.integers(1, 1 << 62)) << int(rng.integers(0, nb // 2))
        g0 = P.Generator.from_seed(spec, int(rng.integers(1 << 32)))
        sub = D.Substreams.from_generator(g0, n, stride=stride, blocks=blocks, block_stride=bstride)
        S = sub.states.cpu().numpy().astype(np.uint64)
        for _ in range(4):
            b, i = int(rng.integers(blocks)), int(rng.integers(n))
            g = g0.clone()
            steps = b * bstride + i * stride
            if steps:
                g.jump(P.compute_jump_poly(spec, steps))
            assert list(g.flat_words()) == [int(v) for v in S[:, b * n + i]], (name, n, blocks, b, i)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SLP_FUZZ_SEEDS", "12")) // 3 + 1))
def test_hwd_counts_fuzz(seed):
    """HWD counting (K6) on random ranges, k, modes and generators against the
    oracle's per-signature counts and weight sums (hwd.py:206-233)."""
    from paper_1805_01407_b200 import hwd

    rng = np.random.default_rng(7000 + seed)
    for _ in range(3):
        split = bool(rng.integers(4) == 0)
        names = [n for n in ALL if P.get_spec(n).kind.w == 64] if split else ALL
        name = names[rng.integers(len(names))]
        spec = P.get_spec(name)
        w = 32 if split else spec.kind.w
        k = int(rng.choice([1, 2, 3, 5, 8, 9, 10]))
        mode = "transitional" if rng.integers(2) else "standard"
        cfg = hwd.HwdConfig(w=w, k=k, mode=mode, split=split)
        c0 = int(rng.integers(k, 5000))
        c1 = c0 + int(rng.integers(1, 200_000))
        seed_g = int(rng.integers(1 << 30))
        ctr = hwd._GpuCounter(spec, seed_g, cfg)
        ctr.count(c0, c1)
        got_c, got_s = ctr.snapshot()
        vals = O.hwd_test_values(name, seed_g, c1, split, mode == "transitional", w)
        want_c, want_s = O.hwd_counts(vals, c0, c1, k, w, cfg.ell)
        msg = f"{name} k={k} {mode} split={split} [{c0}, {c1})"
        np.testing.assert_array_equal(got_c, want_c, err_msg=msg)
        np.testing.assert_array_equal(got_s, want_s, err_msg=msg)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SLP_FUZZ_SEEDS", "12")) // 3 + 1))
def test_split_fuzz(seed):
    """Few long substreams (segment split inside the C ABI) on random
    generators, counts and row lengths: fill, store + checksum and the fused
    checksum against the oracle, with the advanced states."""
    rng = np.random.default_rng(11000 + seed)
    for _ in range(3):
        name = ALL[rng.integers(len(ALL))]
        spec = P.get_spec(name)
        w = spec.kind.w
        n = int(rng.choice([1, 2, 3, 7]))
        T = int(rng.choice([4096, 8192, 3 * 4096, 1 << 15]))
        if D._split_factor(spec, n, T, "stream", T) == 1:
            continue
        flat = rng.integers(0, 1 << 63, size=(spec.kind.k, n), dtype=np.uint64) | np.uint64(1)
        if w == 32:
            flat &= np.uint64(0xFFFFFFFF)
        want, want_S = O.vec_outputs(name, flat, T)
        msg = f"{name} n={n} T={T}"
        sub = D.Substreams.from_states(spec, flat)
        got = D.fill(spec, sub.states, T).cpu().numpy()
        np.testing.assert_array_equal(got.astype(np.uint64), want.astype(np.uint64), err_msg=msg)
        np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S, err_msg=msg)
        oc = O.checksum(want, w)
        c = D.Substreams.from_states(spec, flat).checksum(T, exact=True)
        assert (c.sum, c.xor, c.mant) == (oc["sum"], oc["xor"], oc["mant"]), msg
        sub2 = D.Substreams.from_states(spec, flat)
        _, c2 = D.fill_checksum(spec, sub2.states, T)
        assert (c2.sum, c2.xor, c2.mant) == (oc["sum"], oc["xor"], oc["mant"]), msg
        np.testing.assert_array_equal(sub2.states.cpu().numpy().astype(np.uint64), want_S, err_msg=msg)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SLP_FUZZ_SEEDS", "12")) // 2 + 1))
def test_few_long_split_fuzz(seed):
    """Few, long substreams through the segment split, in every layout the
    split serves: contiguous and padded stream-major rows, position-major
    (incl. unaligned pitch, which falls back to the unsplit paths)."""
    rng = np.random.default_rng(13000 + seed)
    for _ in range(4):
        name = ALL[rng.integers(len(ALL))]
        spec = P.get_spec(name)
        w = spec.kind.w
        n = int(rng.choice([1, 2, 5, 16, 33]))
        T = int(rng.choice([1 << 13, 3 << 12, 1 << 14, 5 << 12]))
        layout = str(rng.choice(["stream", "position"]))
        pad = int(rng.choice([0, 1, 2, 8, 16]))
        flat = rng.integers(0, 1 << 63, size=(spec.kind.k, n), dtype=np.uint64) | np.uint64(1)
        if w == 32:
            flat &= np.uint64(0xFFFFFFFF)
        want, want_S = O.vec_outputs(name, flat, T)
        want = want.astype(np.uint64 if w == 64 else np.uint32)
        if layout == "position":
            want = want.T.copy()
        rows, cols = want.shape
        dt = torch.uint64 if w == 64 else torch.uint32
        big = torch.zeros((rows, cols + pad), dtype=dt, device="cuda")
        sub = D.Substreams.from_states(spec, flat)
        D.fill(spec, sub.states, T, out=big[:, :cols], layout=layout)
        msg = f"{name} n={n} T={T} {layout} pad={pad} J={D._split_factor(spec, n, T, layout, cols + pad)}"
        got = big.cpu().numpy()
        np.testing.assert_array_equal(got[:, :cols], want, err_msg=msg)
        assert not got[:, cols:].any(), msg
        np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S, err_msg=msg)


_SHAPES = [("xoroshiro", 2, 64), ("xoroshiro", 16, 64), ("xoshiro", 4, 64), ("xoshiro", 8, 64),
           ("xorshift", 2, 64), ("xoroshiro", 2, 32), ("xoshiro", 4, 32), ("xoshiro", 8, 32), ("xorshift", 2, 32)]


def _random_custom(rng, tag):
    fam, k, w = _SHAPES[rng.integers(len(_SHAPES))]
    a, b, c = (int(x) for x in rng.integers(1, w, size=3))
    kind = str(rng.choice(["none", "plus", "star", "plusplus", "starstar"]))
    words = [0, k - 1] if (fam == "xoroshiro" and k > 2) else list(range(k))
    i, j = int(rng.choice(words)), int(rng.choice(words))
    odd = lambda: int(rng.integers(1, 1 << (w - 1))) * 2 + 1  # noqa: E731
    kw = {"none": dict(word_i=i), "plus": dict(word_i=i, word_j=j), "star": dict(word_i=i, S=odd()),
          "plusplus": dict(word_i=i, word_j=j, R=int(rng.integers(1, w))),
          "starstar": dict(word_i=i, S=odd(), R=int(rng.integers(1, w)), T=odd())}[kind]
    name = f"fuzz-{tag}"
    spec = P.custom_spec(fam, k, w, a, b, c if fam != "xoshiro" else None,
                         scrambler=P.ScramblerSpec(kind, **kw), name=name)
    sc = spec.scrambler
    O.SPECS[name] = (fam, k, w, (a, b, c if fam != "xoshiro" else None), kind, sc.word_i, sc.word_j, sc.S, sc.R,
                     sc.T)
    return name, spec


@pytest.mark.parametrize("seed", range(int(os.environ.get("SLP_FUZZ_SEEDS", "12")) // 2 + 1))
def test_custom_engine_fuzz(seed):
    """Random custom_spec engines (any parameters, scrambler and word choice)
    through the run-time parameter kernels: fill (both layouts, all kinds)
    and the fused checksum against the oracle."""
    rng = np.random.default_rng(17000 + seed)
    for it in range(4):
        name, spec = _random_custom(rng, f"{seed}-{it}")
        w = spec.kind.w
        n = int(rng.choice([1, 33, 300, 2000]))
        T = int(rng.choice([1, 17, 64, 129, 512, 1000]))
        layout = str(rng.choice(["stream", "position"]))
        kinds = ["native", "f64"] if w == 64 else ["native", "u64", "f32"]
        kind = kinds[rng.integers(len(kinds))]
        flat = rng.integers(0, 1 << 63, size=(spec.kind.k, n), dtype=np.uint64) | np.uint64(1)
        if w == 32:
            flat &= np.uint64(0xFFFFFFFF)
        want, want_S = O.vec_outputs(name, flat, T)
        oc = O.checksum(want, w)
        want = want.astype(np.uint64 if w == 64 else np.uint32)
        if kind == "u64":
            want = want.astype(np.uint64)
        elif kind == "f64":
            want = O.to_f64(want)
        elif kind == "f32":
            want = O.to_f32(want)
        if layout == "position":
            want = want.T.copy()
        msg = f"{spec} n={n} T={T} {layout} {kind}"
        sub = D.Substreams.from_states(spec, flat)
        got = D.fill(spec, sub.states, T, kind=kind, layout=layout).cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint8), want.view(np.uint8), err_msg=msg)
        np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S, err_msg=msg)
        c = D.Substreams.from_states(spec, flat).checksum(T, exact=True)
        assert (c.sum, c.xor, c.mant) == (oc["sum"], oc["xor"], oc["mant"]), msg

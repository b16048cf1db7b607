"""Every fill kind of every generator against the oracle.  The tile
configuration of kernel K2 is chosen per (generator, kind) from a measured
table (csrc/slp_fill_tuning.h), so each combination is its own code path:
store native, store converted (u64 zero-extension / f64 / f32), store +
checksum in one pass.  Sizes exercise several tiles, the rolled sub-block
loop, the pre-wait chunks, the per-lane tail and warps that process more
than one unit of 32 substreams (next-unit state prefetch)."""

import numpy as np
import pytest

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ALL = P.registry_names(include_analysis=True)


def _flat(spec, L, seed):
    rng = np.random.default_rng(seed)
    flat = rng.integers(0, 1 << 63, size=(spec.kind.k, L), dtype=np.uint64) | np.uint64(1)
    if spec.kind.w == 32:
        flat &= np.uint64(0xFFFFFFFF)
    return flat


def _kinds(w):
    return ["native", "f64"] if w == 64 else ["native", "u64", "f32"]


def _convert(ints, kind, w):
    if kind == "native":
        return ints
    if kind == "u64":
        return ints.astype(np.uint64)
    return O.to_f64(ints) if kind == "f64" else O.to_f32(ints)


def _bits(a):
    return a.view(np.uint64) if a.dtype in (np.float64, np.uint64) else a.view(np.uint32)


@pytest.mark.parametrize("name", ALL)
@pytest.mark.parametrize("T", [1000, 2061])
def test_all_kinds_vs_oracle(name, T):
    spec = P.get_spec(name)
    w = spec.kind.w
    flat = _flat(spec, 45, T)
    want, want_S = O.vec_outputs(name, flat, T)
    want = want.astype(np.uint64 if w == 64 else np.uint32)
    oc = O.checksum(want, w)
    for kind in _kinds(w):
        exp = _convert(want, kind, w)
        sub = D.Substreams.from_states(spec, flat)
        got = sub.fill(T, kind=kind).cpu().numpy()
        np.testing.assert_array_equal(_bits(got), _bits(exp), err_msg=f"{name} {kind}")
        np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S)
        # position-major (2-D TMA path for T >= one tile) is the transpose
        sub = D.Substreams.from_states(spec, flat)
        gotp = sub.fill(T, kind=kind, layout="position").cpu().numpy()
        np.testing.assert_array_equal(_bits(gotp), _bits(exp.T.copy()), err_msg=f"{name} {kind} position")
        if kind in ("native", "f64", "f32"):
            sub = D.Substreams.from_states(spec, flat)
            out, c = D.fill_checksum(spec, sub.states, T, kind=kind)
            np.testing.assert_array_equal(_bits(out.cpu().numpy()), _bits(exp), err_msg=f"{name} csum {kind}")
            assert (c.sum, c.xor, c.mant) == (oc["sum"], oc["xor"], oc["mant"]), (name, kind)
            np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoroshiro1024plusplus",
                                  "xoshiro512plusplus", "xoshiro128starstar", "xoroshiro64starstar"])
def test_many_units_per_warp(name):
    """More 32-substream units than resident warps (148 SMs x 7 warps), ragged."""
    spec = P.get_spec(name)
    w = spec.kind.w
    L, T = 148 * 7 * 32 * 2 + 5, 300
    flat = _flat(spec, L, 11)
    want, want_S = O.vec_outputs(name, flat, T)
    want = want.astype(np.uint64 if w == 64 else np.uint32)
    sub = D.Substreams.from_states(spec, flat)
    got = sub.fill(T).cpu().numpy()
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S)
    sub = D.Substreams.from_states(spec, flat)
    np.testing.assert_array_equal(sub.fill(T, layout="position").cpu().numpy(), want.T)
    sub = D.Substreams.from_states(spec, flat)
    _, c = D.fill_checksum(spec, sub.states, T)
    oc = O.checksum(want, w)
    assert (c.sum, c.xor, c.mant) == (oc["sum"], oc["xor"], oc["mant"])


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro1024plusplus", "xoshiro128plusplus",
                                  "xoroshiro64star", "xorshift128plus"])
@pytest.mark.parametrize("T", [31, 32, 33, 64, 100, 127])
def test_short_rows_vs_oracle(name, T):
    """Rows shorter than one tuned tile use the short (256-byte) tile shape."""
    spec = P.get_spec(name)
    w = spec.kind.w
    flat = _flat(spec, 1000, T)
    want, want_S = O.vec_outputs(name, flat, T)
    want = want.astype(np.uint64 if w == 64 else np.uint32)
    for kind in _kinds(w):
        sub = D.Substreams.from_states(spec, flat)
        got = sub.fill(T, kind=kind).cpu().numpy()
        np.testing.assert_array_equal(_bits(got), _bits(_convert(want, kind, w)), err_msg=f"{name} {kind} T={T}")
        np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro1024starstar", "xoshiro128plus"])
@pytest.mark.parametrize("T", [1000, 1151, 300])
def test_ragged_tail_without_state_write_back(name, T):
    """Whole tiles + k_fill_tail, also when the caller does not advance the
    states (the tile kernel then hands the tail its states in a temporary)."""
    spec = P.get_spec(name)
    w = spec.kind.w
    flat = _flat(spec, 77, T)
    want, want_S = O.vec_outputs(name, flat, T)
    want = want.astype(np.uint64 if w == 64 else np.uint32)
    sub = D.Substreams.from_states(spec, flat)
    got = sub.fill(T, advance=False).cpu().numpy()
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), flat)  # untouched
    got2 = sub.fill(T).cpu().numpy()
    np.testing.assert_array_equal(got2, want)
    np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plusplus", "xoroshiro1024star",
                                  "xoshiro128starstar", "xoroshiro64starstar"])
@pytest.mark.parametrize("T,n,pad", [(1055, 1001, 0), (127, 37, 0), (2047, 70, 0), (1026, 33, 0), (1024, 65, 1),
                                     (300, 64, 3), (1151, 3, 0)])
def test_odd_pitch_rows(name, T, n, pad):
    """Stream-major rows whose pitch is not a multiple of 16 bytes (TMA needs
    16-byte aligned row starts, profiles/tma_align_probe.cu) take the staged
    path; tails and short rows included.  Bytes after the last row and in
    the row padding stay untouched."""
    import torch

    spec = P.get_spec(name)
    w = spec.kind.w
    flat = _flat(spec, n, T + n)
    want_i, want_S = O.vec_outputs(name, flat, T)
    for kind in _kinds(w):
        want = _convert(want_i.astype(np.uint64 if w == 64 else np.uint32), kind, w)
        dt = {np.dtype(np.uint64): torch.uint64, np.dtype(np.uint32): torch.uint32,
              np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}[want.dtype]
        ld = T + pad
        flatbuf = torch.zeros(n * ld + 64, dtype=dt, device="cuda")
        out = flatbuf[: n * ld].view(n, ld)[:, :T]
        sub = D.Substreams.from_states(spec, flat)
        D.fill(spec, sub.states, T, out=out, kind=kind)
        got = out.cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint8), want.view(np.uint8), err_msg=f"{name} {kind}")
        np.testing.assert_array_equal(sub.states.cpu().numpy().astype(np.uint64), want_S)
        rest = flatbuf.cpu().numpy()
        assert not rest[n * ld:].view(np.uint8).any()
        if pad:
            assert not rest[: n * ld].reshape(n, ld)[:, T:].view(np.uint8).any()

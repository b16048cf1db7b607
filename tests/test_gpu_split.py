"""Segment split beyond contiguous stream-major rows:
few, long substreams written to PADDED stream-major rows (4-D store map,
segment (i, j) = row i, column j*T/J) and to the POSITION-major layout
(segments in j-major order; 2-D store map when a warp's segments share a row
block, element stores otherwise).  Outputs, untouched padding and advanced
states against the oracle."""

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SENT = 0x5A


def want_outputs(name, S0, T):
    return O.vec_outputs(name, S0.astype(np.uint64), T)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoroshiro1024plusplus",
                                  "xoshiro128starstar"])
@pytest.mark.parametrize("n,T,pad", [(1, 1 << 16, 16), (3, 1 << 15, 32), (16, 1 << 15, 64), (40, 8192, 128)])
def test_padded_stream_major(name, n, T, pad):
    spec = P.get_spec(name)
    es = spec.kind.w // 8
    sub = D.Substreams.from_seed(spec, 11, n)
    S0 = sub.states_numpy()
    assert D._split_factor(spec, n, T, "stream", T + pad) > 1
    dt = torch.uint64 if es == 8 else torch.uint32
    buf = torch.full((n, T + pad), SENT, dtype=dt, device="cuda")
    out = sub.fill(T, out=buf[:, :T])
    assert out.data_ptr() == buf.data_ptr()
    want, want_S = want_outputs(name, S0, T)
    got = buf.cpu().numpy()
    np.testing.assert_array_equal(got[:, :T].astype(np.uint64), want)
    assert (got[:, T:] == SENT).all()  # padding untouched
    np.testing.assert_array_equal(sub.states_numpy().astype(np.uint64), want_S)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoshiro128starstar", "xoroshiro64star"])
@pytest.mark.parametrize("n,T,pad", [(1, 1 << 16, 0), (5, 1 << 15, 0), (5, 1 << 15, 3), (32, 8192, 0),
                                     (64, 8192, 0), (64, 8192, 16)])
@pytest.mark.parametrize("kind", ["native", "float"])
def test_position_major(name, n, T, pad, kind):
    spec = P.get_spec(name)
    w = spec.kind.w
    k = ("f64" if w == 64 else "f32") if kind == "float" else "native"
    sub = D.Substreams.from_seed(spec, 5, n)
    S0 = sub.states_numpy()
    assert D._split_factor(spec, n, T, "position", n + pad) > 1
    dt = {("native", 64): torch.uint64, ("native", 32): torch.uint32, ("f64", 64): torch.float64,
          ("f32", 32): torch.float32}[(k, w)]
    buf = torch.zeros((T, n + pad), dtype=dt, device="cuda")
    buf.view(torch.uint8).fill_(SENT)
    sub.fill(T, out=buf[:, :n], layout="position", kind=k)
    want, want_S = want_outputs(name, S0, T)
    if k == "f64":
        want = O.to_f64(want)
    elif k == "f32":
        want = O.to_f32(want)
    got = buf.cpu().numpy()
    np.testing.assert_array_equal(got[:, :n].view(np.uint8),
                                  np.ascontiguousarray(want.T.astype(got.dtype)).view(np.uint8))
    if pad:
        assert (got[:, n:].view(np.uint8) == SENT).all()
    np.testing.assert_array_equal(sub.states_numpy().astype(np.uint64), want_S)


def test_split_rates_lift_the_cliff():
    """The two shapes that ran at 0.005 TB/s unsplit (profiles/round2_slow_shapes.jsonl)."""
    spec = P.get_spec("xoshiro256starstar")
    sub = D.Substreams.from_seed(spec, 42, 16)
    T = 1 << 22
    buf = torch.empty((16, T + 16), dtype=torch.uint64, device="cuda")
    pm = torch.empty((T, 16), dtype=torch.uint64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for args in (dict(out=buf[:, :T]), dict(out=pm, layout="position")):
        sub.fill(T, **args)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            sub.fill(T, **args)
        e1.record()
        e1.synchronize()
        tbs = 16 * T * 8 * 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
        assert tbs > 0.5, (args.get("layout", "stream"), tbs)


@pytest.mark.parametrize("name,kind", [(n, k) for n in ["xoshiro256starstar", "xoroshiro128plus", "xoroshiro1024starstar",
                                                        "xoshiro128starstar", "xoroshiro64starstar"]
                                       for k in ["native", "float"] + (["u64"] if P.get_spec(n).kind.w == 32 else [])])
@pytest.mark.parametrize("n,T,pad,off", [(225, 70, 0, 0), (1001, 64, 2, 1), (449, 33, 1, 3), (3, 100, 0, 1),
                                         (672, 96, 5, 2), (7, 5, 0, 0)])
def test_position_major_unaligned_rows(name, n, T, pad, off, kind):
    """Rows no TMA map can address (odd pitch / unaligned base): the
    CTA-staged path (k_fill_pos_cta: sector-aligned bulk interiors, element
    stores at the CTA edges) -- partial CTA blocks, partial tiles, padding."""
    spec = P.get_spec(name)
    w = spec.kind.w
    k = ("f64" if w == 64 else "f32") if kind == "float" else kind
    dt = {("native", 64): torch.uint64, ("native", 32): torch.uint32, ("f64", 64): torch.float64,
          ("f32", 32): torch.float32, ("u64", 32): torch.uint64}[(k, w)]
    sub = D.Substreams.from_seed(spec, 9, n)
    S0 = sub.states_numpy()
    ld = n + pad + (1 if (n + pad) % 2 == 0 else 0)  # odd pitch
    flat = torch.empty(T * ld + off + 8, dtype=dt, device="cuda")
    flat.view(torch.uint8).fill_(SENT)
    view = flat[off:off + T * ld].view(T, ld)[:, :n]
    sub.fill(T, out=view, layout="position", kind=k)
    want, want_S = want_outputs(name, S0, T)
    if k == "f64":
        want = O.to_f64(want)
    elif k == "f32":
        want = O.to_f32(want)
    got = flat.cpu().numpy()
    body = got[off:off + T * ld].reshape(T, ld)
    np.testing.assert_array_equal(body[:, :n].view(np.uint8), np.ascontiguousarray(want.T.astype(got.dtype)).view(np.uint8))
    mask = np.ones(got.shape, dtype=bool)
    mask[off:off + T * ld] = False
    inner = np.zeros((T, ld), dtype=bool)
    inner[:, :n] = True
    mask[off:off + T * ld] |= ~inner.reshape(-1)
    assert (got[mask].view(np.uint8) == SENT).all()  # nothing outside the view written
    np.testing.assert_array_equal(sub.states_numpy().astype(np.uint64), want_S)

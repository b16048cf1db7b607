"""custom_spec engines (generators.py:127-135) on the device: the run-time
parameter kernels (GenR<>) behind the same C ABI, against the reference's
outputs for the same custom specs (tests/golden/custom.json) and the oracle."""

import json
import os

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from paper_1805_01407_b200.generators import native_id
from oracle import oracle as O

pytestmark = pytest.mark.gpu

with open(os.path.join(os.path.dirname(__file__), "golden", "custom.json")) as _f:
    CUSTOM = json.load(_f)
DEVICE = [n for n, d in CUSTOM.items() if not (d["family"] == "xoroshiro" and d["k"] in (4, 8))]


def spec_of(name):
    d = CUSTOM[name]
    return P.custom_spec(d["family"], d["k"], d["w"], d["a"], d["b"], d["c"],
                         scrambler=P.ScramblerSpec(**d["scrambler"]), name=name)


def hexs(vs):
    return [hex(int(v)) for v in vs]


@pytest.mark.parametrize("name", DEVICE)
def test_substreams_and_fill(name):
    d = CUSTOM[name]
    spec = spec_of(name)
    assert native_id(spec) >= 1024
    sub = D.Substreams.from_seed(spec, 42, 40)               # K1 (run-time parameters)
    assert [hexs(sub.states[:, i].cpu().numpy()) for i in range(40)] == d["substreams"]
    S0 = sub.states_numpy()
    out = sub.fill(300).cpu().numpy()                         # K2, stream-major TMA path
    assert hexs(out[0, :100]) == d["first_outputs_seed42"]
    want, want_S = O.vec_outputs(name, S0.astype(np.uint64), 300)
    np.testing.assert_array_equal(out.astype(np.uint64), want)
    np.testing.assert_array_equal(sub.states_numpy().astype(np.uint64), want_S)


def kinds_of(w):
    """Output kinds defined for a word width (zero-extended u64 only for w = 32)."""
    return ["native", "f64"] if w == 64 else ["native", "u64", "f32"]


@pytest.mark.parametrize("name,kind", [(n, k) for n in DEVICE for k in kinds_of(CUSTOM[n]["w"])])
@pytest.mark.parametrize("layout", ["stream", "position"])
def test_fill_kinds_layouts(name, kind, layout):
    spec = spec_of(name)
    rng = np.random.default_rng(len(name))
    n, T = int(rng.integers(33, 300)), int(rng.integers(17, 700))
    sub = D.Substreams.from_seed(spec, 7, n)
    S0 = sub.states_numpy().astype(np.uint64)
    got = sub.fill(T, kind=kind, layout=layout).cpu().numpy()
    want, _ = O.vec_outputs(name, S0, T)
    if kind == "f64":
        want = O.to_f64(want)
    elif kind == "f32":
        want = O.to_f32(want)
    if layout == "position":
        want = want.T
    np.testing.assert_array_equal(got.view(np.uint8), np.ascontiguousarray(want.astype(got.dtype)).view(np.uint8))


@pytest.mark.parametrize("name", DEVICE)
def test_fused_and_store_checksum(name):
    spec = spec_of(name)
    sub = D.Substreams.from_seed(spec, 42, 3000)
    S0 = sub.states_numpy().astype(np.uint64)
    want, _ = O.vec_outputs(name, S0, 512)
    oc = O.checksum(want, spec.kind.w)
    c = D.Substreams.from_states(spec, S0).checksum(512, f64=True)   # K4
    assert (c.sum, c.xor, c.mant) == (oc["sum"], oc["xor"], oc["mant"])
    assert abs(c.fsum_f64 - c.fsum) <= 1e-12 * abs(c.fsum)
    out2, c2 = D.fill_checksum(spec, D.Substreams.from_states(spec, S0).states, 512)
    np.testing.assert_array_equal(out2.cpu().numpy().astype(np.uint64), want)
    assert (c2.sum, c2.xor, c2.mant) == (oc["sum"], oc["xor"], oc["mant"])


@pytest.mark.parametrize("name", DEVICE)
def test_output_stream_and_laned(name):
    d = CUSTOM[name]
    spec = spec_of(name)
    vals = np.concatenate(list(P.output_stream(spec, 42, 3000, lanes=5, lane_len=512)))
    assert hexs(vals) == d["laned_3000"]
    # one long substream: the C ABI's segment split (K1 segments + K2)
    one = D.Substreams.from_seed(spec, 42, 1)
    long_out = one.fill(1 << 14).cpu().numpy()
    want, _ = O.vec_outputs(name, np.array([[int(x, 16)] for x in d["substreams"][0]], dtype=np.uint64), 1 << 14)
    np.testing.assert_array_equal(long_out.astype(np.uint64), want)


@pytest.mark.parametrize("name", DEVICE)
def test_vecstepper(name):
    d = CUSTOM[name]
    spec = spec_of(name)
    from paper_1805_01407_b200.engines import VecStepper

    st = VecStepper(spec.kind, spec.params)
    S = np.array([[int(x, 16) for x in lane] for lane in d["substreams"]], dtype=np.uint64).T.copy()
    for _ in range(64):
        st.step(S)                                  # the reference's numpy (k, L) arrays
    assert [hexs(st.flat(S)[:, i]) for i in range(40)] == d["substreams_after_64"]
    Sd = torch.from_numpy(np.array([[int(x, 16) for x in lane] for lane in d["substreams"]], dtype=np.uint64).T
                          .copy().astype(np.uint64 if spec.kind.w == 64 else np.uint32)).cuda()
    st.advance(Sd, 64)                              # K1 jump by x^64
    assert [hexs(Sd[:, i].cpu().numpy()) for i in range(40)] == d["substreams_after_64"]


def test_unsupported_shape_raises():
    spec = spec_of("xoroshiro256-4w")
    g = P.Generator.from_seed(spec, 42)             # host path works
    assert hex(g.next()) == CUSTOM["xoroshiro256-4w"]["first_outputs_seed42"][0]
    with pytest.raises(ValueError, match="unsupported"):
        D.Substreams.from_seed(spec, 42, 4)

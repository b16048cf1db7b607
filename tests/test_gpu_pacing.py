"""Store pacing (slp_set_fill_pace) only delays tile stores: paced and
unpaced fills write identical bytes, in every TMA store mode (stream-major,
row-group for odd pitch, position-major), with the checksum fused and with
the segment split, and against the oracle."""

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def paced():
    prev = D.set_fill_pace(None)
    yield
    D.set_fill_pace(prev)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoshiro128plusplus",
                                  "xoroshiro1024starstar"])
@pytest.mark.parametrize("gbps", [0, 500, 6500])
def test_paced_fill_equals_oracle(paced, name, gbps):
    spec = P.get_spec(name)
    n, T = 3 * 32 * 7 + 5, 1024
    sub = D.Substreams.from_seed(spec, 42, n)
    S0 = sub.states.cpu().numpy().astype(np.uint64)
    want, _ = O.vec_outputs(name, S0, T)
    D.set_fill_pace(gbps)
    for layout in ("stream", "position"):
        got = D.Substreams.from_states(spec, S0).fill(T, layout=layout).cpu().numpy()
        np.testing.assert_array_equal(got, want if layout == "stream" else want.T, err_msg=f"{layout} {gbps}")
    # odd row pitch: the row-group TMA path
    ld = T + 1
    dt = torch.uint64 if spec.kind.w == 64 else torch.uint32
    buf = torch.zeros((n, ld), dtype=dt, device="cuda")
    D.Substreams.from_states(spec, S0).fill(T, out=buf[:, :T])
    np.testing.assert_array_equal(buf[:, :T].cpu().numpy(), want)
    # store + checksum in one pass
    out, c = D.fill_checksum(spec, D.Substreams.from_states(spec, S0).states, T)
    np.testing.assert_array_equal(out.cpu().numpy(), want)
    oc = O.checksum(want, spec.kind.w)
    assert (c.sum, c.xor) == (oc["sum"], oc["xor"])


def test_paced_split_fill_equals_unpaced(paced):
    spec = P.get_spec("xoshiro256starstar")
    sub = D.Substreams.from_seed(spec, 7, 3)
    S0 = sub.states.clone()
    D.set_fill_pace(0)
    a = D.fill(spec, S0.clone(), 1 << 16)
    D.set_fill_pace(6500)
    b = D.fill(spec, S0.clone(), 1 << 16)
    assert torch.equal(a, b)

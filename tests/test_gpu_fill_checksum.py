"""Store + checksum in one pass (slp_fill_checksum) against the separate
fill and the reference's golden checksums (config 3 at reduced size)."""

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key,kind", [("c3s/xoroshiro128plus", "f64"), ("c3s/xoroshiro128plusplus", "native"),
                                      ("c2s/xoshiro256starstar", "f64"), ("c4s/xoshiro128starstar", "f32"),
                                      ("c5s/xoroshiro1024starstar", "native")])
def test_fill_checksum_matches_golden(G, key, kind):
    g = G("checksums_small")[key]
    spec = P.get_spec(g["name"])
    sub = D.Substreams.from_seed(spec, g["seed"], g["substreams"], blocks=g["blocks"])
    ref = D.Substreams.from_seed(spec, g["seed"], g["substreams"], blocks=g["blocks"])
    out, c = D.fill_checksum(spec, sub.states, g["T"], kind=kind)
    assert hex(c.sum) == g["sum"] and hex(c.xor) == g["xor"] and hex(c.mant) == g["mant"]
    assert float.hex(c.fsum) == g["fsum"]
    want = ref.fill(g["T"], kind=kind)
    assert torch.equal(out, want)
    assert torch.equal(sub.states, ref.states)


def test_fill_checksum_ragged_and_fallback():
    spec = P.get_spec("xoshiro256plusplus")
    rng = np.random.default_rng(4)
    flat = rng.integers(1, 1 << 63, size=(4, 77), dtype=np.uint64)
    want, _ = O.vec_outputs("xoshiro256plusplus", flat, 1000)
    oc = O.checksum(want, 64)
    sub = D.Substreams.from_states(spec, flat)
    out, c = D.fill_checksum(spec, sub.states, 1000)            # ragged n and T: TMA path + tails
    np.testing.assert_array_equal(out.cpu().numpy(), want)
    assert (c.sum, c.xor, c.mant) == (oc["sum"], oc["xor"], oc["mant"])
    sub2 = D.Substreams.from_states(spec, flat)
    big = torch.empty((77, 1003), dtype=torch.uint64, device="cuda")
    out2, c2 = D.fill_checksum(spec, sub2.states, 20, out=big[:, 1:21])  # unaligned: K4 + K2 fallback
    np.testing.assert_array_equal(out2.cpu().numpy(), want[:, :20])
    o20 = O.checksum(want[:, :20], 64)
    assert (c2.sum, c2.xor, c2.mant) == (o20["sum"], o20["xor"], o20["mant"])

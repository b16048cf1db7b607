"""BASELINE configs 1, 3 and 4 in STORE mode at full size.

Config 3: 2^21 substreams x 1024 outputs -> 2^31 float64 (16 GiB); config 4:
2^22 x 1024 -> 2^32 uint32 / float32 (16 GiB each), i.e. exactly where a
32-bit element index would overflow.  The stored bytes are reduced on the
device independently of the kernels' own checksum code and compared with the
reference's full-size checksums (tests/golden/checksums_big.json = SURVEY
Appendix A, made by tests/golden/make_golden.py from the reference):

* integer store: wrapping sum and xor == golden ``sum`` / ``xor``;
* float store: every element equals the conversion of the stored integer
  (f64: f * 2^53 == x >> 11, generators.py:307-311; f32: f * 2^24 == x >> 8),
  and the exact integer sum of f * 2^53 (f * 2^24) == golden ``mant``;
* sampled rows (first, last, warp and TMA-box edges, random) == the oracle's
  scalar outputs of substream i = seed * M^(i * 2^(n/2)) (generators.py:315-334);
* store + checksum in one pass (slp_fill_checksum) == golden, same bytes.
"""

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1
CHUNK = 1 << 28


def _xor_reduce(t):
    acc = 0
    while t.numel() > 1:
        if t.numel() & 1:
            acc ^= int(t[-1].item())
            t = t[:-1]
        h = t.numel() // 2
        t = t[:h] ^ t[h:]
    if t.numel():
        acc ^= int(t[0].item())
    return acc


def int_sum_xor(out, w):
    """Exact sum (mod 2^64) and xor of stored w-bit integers, on the device."""
    v = out.reshape(-1).view(torch.int64 if w == 64 else torch.int32)
    s, x = 0, 0
    for c in v.split(CHUNK):
        c64 = c.to(torch.int64) & 0xFFFFFFFF if w == 32 else c
        lo = int((c64 & 0xFFFFFFFF).sum().item())
        hi = int(((c64 >> 32) & 0xFFFFFFFF).sum().item())
        s = (s + (hi << 32) + lo) & M64
        x ^= _xor_reduce(c) & ((1 << w) - 1)
    return s, x


def float_mant_and_match(fout, iout, w):
    """Exact sum of f * 2^53 (2^24) and elementwise f <-> conversion of the
    stored integer x (f64: x >> 11, f32: x >> 8)."""
    shift, scale = (11, 2.0 ** 53) if w == 64 else (8, 2.0 ** 24)
    fv = fout.reshape(-1)
    iv = iout.reshape(-1).view(torch.int64 if w == 64 else torch.int32)
    mant = 0
    for f, x in zip(fv.split(CHUNK), iv.split(CHUNK)):
        m = (f.to(torch.float64) * scale).to(torch.int64)
        xi = x.to(torch.int64) & 0xFFFFFFFF if w == 32 else x
        want = (xi >> shift) & ((1 << (64 - shift)) - 1)  # logical shift of the unsigned word
        assert torch.equal(m, want), "float store != conversion of the integer store"
        mant += (int((m >> 26).sum().item()) << 26) + int((m & ((1 << 26) - 1)).sum().item())
    return mant


def check_rows(name, seed, out, rows, T, w):
    spec = P.get_spec(name)
    J = 1 << (spec.kind.n // 2)
    base = O.seed_flat(name, seed)
    mask = (1 << w) - 1
    for i in rows:
        flat = O.jump(name, base, O.jump_poly(name, i * J)) if i else base
        want, _ = O.outputs(name, flat, T)
        got = out[i].cpu().numpy().view(np.uint64 if w == 64 else np.uint32)
        assert [int(v) for v in got] == [v & mask for v in want], f"substream {i}"


def sample_rows(n, seed):
    rng = np.random.default_rng(seed)
    return sorted({0, 1, 31, 32, 33, 1023, 1024, n // 2, n - 33, n - 2, n - 1,
                   *[int(r) for r in rng.integers(0, n, 6)]})


CONFIG3 = ["xoroshiro128plus", "xoroshiro128plusplus", "xoroshiro128starstar"]
CONFIG4 = ["xoshiro128starstar", "xoshiro128plusplus", "xoroshiro64star", "xoroshiro64starstar"]


@pytest.mark.parametrize("cfg,name", [("c3", n) for n in CONFIG3] + [("c4", n) for n in CONFIG4])
def test_store_full_size(G, cfg, name):
    g = G("checksums_big")[f"{cfg}/{name}"]
    spec = P.get_spec(name)
    w = spec.kind.w
    n, T = g["substreams"], g["T"]
    assert g["blocks"] == 1 and n * T == (1 << 31 if w == 64 else 1 << 32)
    fkind = "f64" if w == 64 else "f32"
    sub = D.Substreams.from_seed(spec, g["seed"], n)
    states0 = sub.states.clone()
    iout = sub.fill(T, advance=False)                    # native integers, 16 GiB
    s, x = int_sum_xor(iout, w)
    assert (hex(s), hex(x)) == (g["sum"], g["xor"])
    check_rows(name, g["seed"], iout, sample_rows(n, len(name)), T, w)
    fout = sub.fill(T, kind=fkind, advance=False)        # converted floats, 16 GiB
    mant = float_mant_and_match(fout, iout, w)
    assert hex(mant) == g["mant"]
    del iout
    torch.cuda.empty_cache()
    # store + checksum in one pass: same bytes, checksum == golden, states advanced
    st = states0.clone()
    out2, c = D.fill_checksum(spec, st, T, kind=fkind)
    assert (hex(c.sum), hex(c.xor), hex(c.mant)) == (g["sum"], g["xor"], g["mant"])
    assert float.hex(c.fsum) == g["fsum"]
    assert torch.equal(out2.view(torch.uint8), fout.view(torch.uint8))
    assert torch.equal(sub.states, states0)  # fill(advance=False) left the states alone
    ref = states0.clone()
    D.fused_checksum(spec, ref, T, exact=False)  # K4 advances its own copy by T steps
    assert torch.equal(st, ref)
    del out2, fout
    torch.cuda.empty_cache()


def test_config1_jump_then_1024_outputs(G):
    """Config 1, second half: jump() once, then 2^10 outputs — all 1024 golden
    values, through the device substream path, the host Generator and the
    laned bulk API fed with the jumped generator (generators.py:315-334, 426-490)."""
    want = G("generators")["xoshiro256starstar"]["jump_outputs_seed42"]
    assert len(want) == 1024
    spec = P.get_spec("xoshiro256starstar")
    dev = D.Substreams.from_seed(spec, 42, 2).fill(1024)[1].cpu().numpy()
    assert [hex(int(v)) for v in dev] == want
    g = P.Generator.from_seed(spec, 42)
    g.jump(P.default_jumps(spec)[0])
    laned = np.concatenate(list(P.LanedStream(spec, generator=g.clone(), lanes=8, lane_len=128).chunks(1024)))
    assert [hex(int(v)) for v in laned] == want
    assert [hex(g.next()) for _ in range(1024)] == want

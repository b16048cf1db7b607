"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Bit-exact for all integer and converted-float
outputs; float64 in-kernel sums within 1e-12 relative (north_star)."""

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ALL = P.registry_names(include_analysis=True)


def hexs(vals):
    return [hex(int(v)) for v in vals]


def flat_np(name, states):
    return states.cpu().numpy().astype(np.uint64)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoroshiro128plusplus",
                                  "xoshiro512starstar", "xoroshiro1024starstar", "xoshiro128starstar",
                                  "xoroshiro64star"])
def test_init_substreams_dense(G, name):
    d = G("substreams")[name]
    sub = D.Substreams.from_seed(P.get_spec(name), d["seed"], 64)
    S = flat_np(name, sub.states)
    for i in range(64):
        assert hexs(S[:, i]) == d["dense_states"][i], i


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoshiro128starstar",
                                  "xoroshiro64star", "xoshiro512starstar"])
def test_init_substreams_sparse(G, name):
    d = G("substreams")[name]
    spec = P.get_spec(name)
    n = (1 << 20) if spec.kind.w == 64 else (1 << 22)
    sub = D.Substreams.from_seed(spec, d["seed"], n)
    S = sub.states
    for idx, want in d["sparse_states"].items():
        i = int(idx)
        if i < n:
            assert hexs(S[:, i].cpu().numpy()) == want, idx


@pytest.mark.parametrize("name", ["xoshiro512starstar", "xoroshiro1024starstar", "xoshiro256starstar"])
def test_long_jump_blocks(G, name):
    d = G("substreams")[name]
    spec = P.get_spec(name)
    sub = D.Substreams.from_seed(spec, d["seed"], 3, blocks=8)
    S = flat_np(name, sub.states)
    for b in range(1, 8):
        assert hexs(S[:, b * 3]) == d["long_jump_blocks"][str(b)]


@pytest.mark.parametrize("name", ALL)
def test_fill_stream_major_matches_scalar(G, name):
    """Stream 0 = Generator.from_seed(42); stream 1 = jumped once (generators.py:315-334)."""
    spec = P.get_spec(name)
    d = G("generators")[name]
    sub = D.Substreams.from_seed(spec, 42, 37)
    out = sub.fill(100)
    assert hexs(out[0].cpu().numpy()) == d["first_outputs_seed42"]
    assert hexs(sub.states[:, 0].cpu().numpy()) == d["state_after_100_seed42"]
    want_j = d["jump_outputs_seed42"][:32]
    out2 = D.Substreams.from_seed(spec, 42, 2).fill(32)
    assert hexs(out2[1].cpu().numpy()) == want_j


@pytest.mark.parametrize("name", ALL)
@pytest.mark.parametrize("T", [1, 15, 16, 33, 257, 1024])
def test_fill_vs_oracle_ragged(name, T):
    """Every substream, ragged stream count and lengths (tails, partial TMA boxes)."""
    spec = P.get_spec(name)
    rng = np.random.default_rng(T)
    L = 45
    k, w = spec.kind.k, spec.kind.w
    flat = rng.integers(0, 1 << 63, size=(k, L), dtype=np.uint64) | np.uint64(1)
    if w == 32:
        flat &= np.uint64(0xFFFFFFFF)
    want, want_S = O.vec_outputs(name, flat, T)
    sub = D.Substreams.from_states(spec, flat)
    got = sub.fill(T).cpu().numpy().astype(np.uint64)
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(flat_np(name, sub.states), want_S)
    # position-major layout is the transpose
    sub2 = D.Substreams.from_states(spec, flat)
    gotp = sub2.fill(T, layout="position").cpu().numpy().astype(np.uint64)
    np.testing.assert_array_equal(gotp, want.T)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoroshiro1024plusplus",
                                  "xoshiro512plus"])
def test_f64_bit_exact(name):
    spec = P.get_spec(name)
    sub = D.Substreams.from_seed(spec, 42, 100)
    ints = D.Substreams.from_seed(spec, 42, 100).fill(300).cpu().numpy()
    f = sub.fill(300, kind="f64").cpu().numpy()
    np.testing.assert_array_equal(f.view(np.uint64), O.to_f64(ints).view(np.uint64))
    assert f.min() >= 0.0 and f.max() < 1.0


def test_f64_matches_next_double(G):
    spec = P.get_spec("xoshiro256starstar")
    f = D.Substreams.from_seed(spec, 42, 1).fill(16, kind="f64").cpu().numpy()[0]
    assert [float.hex(float(x)) for x in f] == G("generators")["xoshiro256starstar"]["first_doubles_seed42"]


@pytest.mark.parametrize("name", ["xoshiro128starstar", "xoshiro128plusplus", "xoroshiro64star",
                                  "xoroshiro64starstar"])
def test_f32_and_u64_kinds(name):
    spec = P.get_spec(name)
    ints = D.Substreams.from_seed(spec, 7, 70).fill(200).cpu().numpy()
    f = D.Substreams.from_seed(spec, 7, 70).fill(200, kind="f32").cpu().numpy()
    np.testing.assert_array_equal(f.view(np.uint32), O.to_f32(ints).view(np.uint32))
    u = D.Substreams.from_seed(spec, 7, 70).fill(200, kind="u64").cpu().numpy()
    np.testing.assert_array_equal(u, ints.astype(np.uint64))
    with pytest.raises(ValueError):
        D.Substreams.from_seed(spec, 7, 4).fill(8, kind="f64")


def test_unaligned_pitch_uses_staged_path():
    spec = P.get_spec("xoshiro256plusplus")
    flat_sub = D.Substreams.from_seed(spec, 42, 50)
    ref = D.Substreams.from_seed(spec, 42, 50).fill(130).cpu().numpy()
    big = torch.zeros((50, 133), dtype=torch.uint64, device="cuda")
    view = big[:, 1:131]  # row pitch 133 elements, base not 16-byte aligned
    D.fill(spec, flat_sub.states, 130, out=view)
    np.testing.assert_array_equal(view.cpu().numpy(), ref)
    assert int(big[:, 0].cpu().numpy().max()) == 0 and int(big[:, 131:].cpu().numpy().max()) == 0


@pytest.mark.parametrize("key", ["c2s/xoshiro256plus", "c2s/xoshiro256plusplus", "c2s/xoshiro256starstar",
                                 "c3s/xoroshiro128plus", "c3s/xoroshiro128plusplus", "c3s/xoroshiro128starstar",
                                 "c4s/xoshiro128starstar", "c4s/xoshiro128plusplus", "c4s/xoroshiro64star",
                                 "c4s/xoroshiro64starstar", "c5s/xoshiro512starstar", "c5s/xoshiro512plusplus",
                                 "c5s/xoroshiro1024starstar", "c5s/xoroshiro1024plusplus"])
def test_fused_small_configs(G, key):
    g = G("checksums_small")[key]
    spec = P.get_spec(g["name"])
    sub = D.Substreams.from_seed(spec, g["seed"], g["substreams"], blocks=g["blocks"])
    c = sub.checksum(g["T"], f64=True)
    assert hex(c.sum) == g["sum"] and hex(c.xor) == g["xor"] and hex(c.mant) == g["mant"]
    assert float.hex(c.fsum) == g["fsum"]
    assert abs(c.fsum_f64 - c.fsum) <= 1e-12 * abs(c.fsum)
    assert c.count == g["blocks"] * g["substreams"] * g["T"]


@pytest.mark.parametrize("key", ["c2/xoshiro256plus", "c2/xoshiro256plusplus", "c2/xoshiro256starstar",
                                 "c3/xoroshiro128plus", "c3/xoroshiro128plusplus", "c3/xoroshiro128starstar",
                                 "c4/xoshiro128starstar", "c4/xoshiro128plusplus", "c4/xoroshiro64star",
                                 "c4/xoroshiro64starstar", "c5/xoshiro512starstar", "c5/xoshiro512plusplus",
                                 "c5/xoroshiro1024starstar", "c5/xoroshiro1024plusplus"])
def test_fused_full_size_configs(G, key):
    """BASELINE configs 2-5 at full size: checksums equal the reference's."""
    g = G("checksums_big").get(key)
    if g is None:
        pytest.skip("golden checksum not generated")
    spec = P.get_spec(g["name"])
    sub = D.Substreams.from_seed(spec, g["seed"], g["substreams"], blocks=g["blocks"])
    c = sub.checksum(g["T"], f64=True)
    assert hex(c.sum) == g["sum"] and hex(c.xor) == g["xor"] and hex(c.mant) == g["mant"]
    assert float.hex(c.fsum) == g["fsum"]
    assert abs(c.fsum_f64 - c.fsum) <= 1e-12 * abs(c.fsum)


def test_store_equals_fused_full_config2(G):
    """Config 2 store mode (8 GiB): the stored outputs reduce to the reference checksum."""
    g = G("checksums_big").get("c2/xoshiro256starstar")
    if g is None:
        pytest.skip("golden checksum not generated")
    spec = P.get_spec("xoshiro256starstar")
    sub = D.Substreams.from_seed(spec, 42, 1 << 20)
    out = sub.fill(1024)
    v = out.view(torch.int64)
    s = int(v.sum(dtype=torch.int64).item()) & ((1 << 64) - 1)  # wraps mod 2^64
    x = v[:, 0].clone()
    cols = v
    while cols.shape[1] > 1:
        h = cols.shape[1] // 2
        cols = cols[:, :h] ^ cols[:, h:2 * h]
    xr = cols[:, 0]
    while xr.numel() > 1:
        h = xr.numel() // 2
        xr = xr[:h] ^ xr[h:2 * h]
    del x
    assert hex(s) == g["sum"]
    assert hex(int(xr.item()) & ((1 << 64) - 1)) == g["xor"]


@pytest.mark.parametrize("key", ["xoroshiro128plus/5/2500/6/128", "xoshiro256starstar/5/2500/6/128",
                                 "xoroshiro1024plusplus/5/2500/6/128", "xorshift128/5/2500/6/128",
                                 "xoshiro128plus/5/2500/6/128", "xoshiro256plus/8/700/1/256",
                                 "xoshiro256starstar/42/5000/4/1000", "xoroshiro64starstar/3/3000/5/256",
                                 "xoshiro512plusplus/11/4096/8/128"])
def test_output_stream_matches_reference(G, key):
    d = G("laned")[key]
    spec = P.get_spec(d["name"])
    chunks = list(P.output_stream(spec, seed=d["seed"], total_values=d["total"], lanes=d["lanes"],
                                  lane_len=d["lane_len"]))
    assert [c.size for c in chunks] == d["chunk_sizes"]
    assert all(c.dtype == np.uint64 for c in chunks)
    assert hexs(np.concatenate(chunks)) == d["values"]


def test_output_stream_config1(G):
    """Config 1: xoshiro256** seed 42, 2^20 outputs through the laned bulk API."""
    spec = P.get_spec("xoshiro256starstar")
    vals = np.concatenate(list(P.output_stream(spec, seed=42, total_values=1 << 20)))
    assert vals.size == 1 << 20
    assert hex(int(vals[0])) == "0x15780b2e0c2ec716"
    assert hex(int(vals[-1])) == "0x6569564c7df21f30"
    c = O.checksum(vals, 64)
    assert hex(c["sum"]) == "0x89f6597c294a86e6" and hex(c["xor"]) == "0x40c711d84f637bcc"


def test_jump_states_matches_host(G):
    spec = P.get_spec("xoroshiro1024plusplus")
    sub = D.Substreams.from_seed(spec, 42, 9)
    before = flat_np("x", sub.states)
    jp = P.compute_jump_poly(spec, 123456789)
    sub.jump(jp)
    after = flat_np("x", sub.states)
    for i in range(9):
        g = P.Generator(spec, [int(v) for v in before[:, i]], ptr=spec.kind.k - 1)
        g.jump(jp)
        assert list(g.flat_words()) == [int(v) for v in after[:, i]]


def test_errors():
    spec = P.get_spec("xoshiro256plus")
    with pytest.raises(ValueError):
        D.Substreams.from_seed(P.custom_spec("xoroshiro", 2, 5, 1, 3, 1), 1, 4)
    sub = D.Substreams.from_seed(spec, 1, 4)
    with pytest.raises(ValueError):
        sub.jump(P.compute_jump_poly(P.get_spec("xoroshiro128"), 5))
    with pytest.raises(ValueError):
        sub.fill(4, kind="f32")


@pytest.mark.parametrize("name", ["xoroshiro128plus", "xoshiro256starstar", "xoshiro512plusplus",
                                  "xoroshiro1024plus", "xorshift128plus", "xoroshiro64starstar",
                                  "xoshiro128plusplus"])
def test_vecstepper_matches_scalar_step(name):
    """test_engines.py:111-136 on the device stepper: 64 steps x 5 lanes."""
    import random

    spec = P.get_spec(name)
    kind, params = spec.kind, spec.params
    rng = random.Random(3)
    states = [P.bits_to_words(rng.randrange(1, 1 << kind.n), kind.k, kind.w) for _ in range(5)]
    npdt = np.uint64 if kind.w == 64 else np.uint32
    S = torch.from_numpy(np.array(list(zip(*states)), dtype=npdt)).cuda()
    st = D.VecStepper(kind, params)
    scalars = [tuple(s) for s in states]
    for _ in range(64):
        scalars = [P.step(kind, params, s) for s in scalars]
        st.step(S)
        got = S.cpu().numpy()
        for j in range(5):
            assert [int(st.word(got, i)[j]) for i in range(kind.k)] == list(scalars[j])
    # advance == repeated steps
    S2 = torch.from_numpy(np.array(list(zip(*states)), dtype=npdt)).cuda()
    st.advance(S2, 64)
    np.testing.assert_array_equal(S2.cpu().numpy(), S.cpu().numpy())


# ---------------------------------------------------------------- edge cases


def test_edge_empty_and_degenerate():
    spec = P.get_spec("xoshiro256starstar")
    sub = D.Substreams.from_seed(spec, 42, 5)
    before = sub.states.clone()
    out = sub.fill(0)
    assert tuple(out.shape) == (5, 0)
    assert torch.equal(sub.states, before)          # T = 0 leaves the states alone
    st = torch.empty((4, 0), dtype=torch.uint64, device="cuda")
    assert tuple(D.fill(spec, st, 16).shape) == (0, 16)   # no substreams
    c = sub.checksum(0)
    assert (c.sum, c.xor, c.mant, c.count) == (0, 0, 0, 0)
    one = D.Substreams.from_seed(spec, 42, 1)        # a single substream = the scalar generator
    g = P.Generator.from_seed(spec, 42)
    assert [int(x) for x in one.fill(70).cpu().numpy()[0]] == [g.next() for _ in range(70)]


def test_edge_zero_base_state_rejected():
    spec = P.get_spec("xoshiro256plus")
    # stride 0 is legal (every substream is the base state) ...
    s0 = D.Substreams.from_generator(P.Generator(spec, [0, 0, 0, 1]), 4, stride=0)
    assert all(int(x) == 1 for x in s0.states[3].cpu().numpy())
    # ... but an all-zero base state is not (generators.py:202-203)
    import ctypes

    from paper_1805_01407_b200 import _native
    base = (ctypes.c_uint64 * 4)(0, 0, 0, 0)
    steps = (ctypes.c_uint64 * 1)(1)
    buf = torch.empty((4, 4), dtype=torch.uint64, device="cuda")
    rc = _native.lib().slp_init_substreams(6, base, 1, steps, 1, ctypes.c_void_p(buf.data_ptr()), 4, 4, None)
    assert rc == _native.SLP_ERR_ZERO_STATE


def test_edge_long_single_stream_and_many_blocks():
    """One substream x 2^22 outputs (ragged vs every tile size) and 20 long-jump blocks (> one K1 batch)."""
    spec = P.get_spec("xoroshiro128plusplus")
    sub = D.Substreams.from_seed(spec, 3, 1)
    T = (1 << 22) + 13
    out = sub.fill(T).cpu().numpy()[0]
    want = O.laned_stream("xoroshiro128plusplus", 3, T, 64, 1 << 16)
    np.testing.assert_array_equal(out, want)
    spec5 = P.get_spec("xoshiro512plusplus")
    many = D.Substreams.from_seed(spec5, 42, 2, blocks=20)
    S = many.states.cpu().numpy()
    g = P.Generator.from_seed(spec5, 42)
    lj = P.default_jumps(spec5)[1]
    for b in range(20):
        assert list(g.flat_words()) == [int(x) for x in S[:, 2 * b]], b
        g.jump(lj)


def test_edge_jump_identity_and_advance_matches_fill():
    spec = P.get_spec("xoroshiro1024star")
    a = D.Substreams.from_seed(spec, 7, 33)
    b = D.Substreams.from_seed(spec, 7, 33)
    a.jump(P.compute_jump_poly(spec, 0))             # x^0 = 1: identity
    assert torch.equal(a.states, b.states)
    a.jump(P.compute_jump_poly(spec, 1000))          # jump 1000 == emit 1000 outputs
    b.fill(1000)
    assert torch.equal(a.states, b.states)


@pytest.mark.parametrize("lanes,lane_len,total", [(1, 7, 100), (3, 1, 10), (5, 1000, 12345), (64, 256, 16384)])
def test_edge_laned_geometries(lanes, lane_len, total):
    spec = P.get_spec("xoshiro128starstar")
    got = np.concatenate(list(P.output_stream(spec, seed=11, total_values=total, lanes=lanes, lane_len=lane_len)))
    g = P.Generator.from_seed(spec, 11)
    assert [int(x) for x in got] == [g.next() for _ in range(total)]


@pytest.mark.parametrize("name,n,T", [("xoshiro256starstar", 1, 1 << 20), ("xoroshiro128plus", 3, 1 << 19),
                                      ("xoshiro128plusplus", 17, 1 << 16), ("xoroshiro1024starstar", 2, 1 << 20)])
def test_segment_split_fill_is_transparent(name, n, T):
    """Few, long substreams are split into jumped segments on the device; the
    output and the advanced states must equal the unsplit computation."""
    import os

    spec = P.get_spec(name)
    assert D._split_factor(spec, n, T, "stream", T) > 1
    a = D.Substreams.from_seed(spec, 5, n)
    out = a.fill(T)
    ref = D.Substreams.from_seed(spec, 5, n)
    want = torch.empty_like(out)
    L = __import__("paper_1805_01407_b200._native", fromlist=["x"])
    import ctypes
    os.environ["SLP_SPLIT"] = "0"  # the unsplit fill: one thread per substream
    try:
        rc = L.lib().slp_fill(D.native_id(spec), ctypes.c_void_p(ref.states.data_ptr()),
                              ctypes.c_void_p(ref.states.data_ptr()), n, n, T, 0, 0,
                              ctypes.c_void_p(want.data_ptr()), T, None)
    finally:
        del os.environ["SLP_SPLIT"]
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    assert torch.equal(a.states, ref.states)


@pytest.mark.parametrize("name,n,T", [("xoshiro256starstar", 1, 1 << 20), ("xoroshiro1024plusplus", 3, 1 << 18),
                                      ("xoshiro128starstar", 5, 1 << 17)])
def test_segment_split_checksums_are_transparent(name, n, T):
    """Few long substreams: the fused checksum (K4) and store + checksum (K2)
    reduce over the segments of the split (inside the C ABI).  Exact fields
    and the advanced states must equal the unsplit K4 pass (SLP_SPLIT=0;
    float64 sum: same set, other order)."""
    import ctypes

    from paper_1805_01407_b200 import _native

    spec = P.get_spec(name)
    assert D._split_factor(spec, n, T, "stream", T) > 1
    ref = D.Substreams.from_seed(spec, 9, n)
    res = torch.empty(_native.CHECKSUM_BYTES, dtype=torch.uint8, device="cuda")
    ws = D._workspace(D.native_id(spec), ref.states.device)
    flags = _native.FUSE_INT | _native.FUSE_EXACT | _native.FUSE_F64
    import os

    os.environ["SLP_SPLIT"] = "0"  # the unsplit K4 pass: one thread per substream
    try:
        rc = _native.lib().slp_fused(D.native_id(spec), ctypes.c_void_p(ref.states.data_ptr()),
                                     ctypes.c_void_p(ref.states.data_ptr()), n, n, T, flags,
                                     ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                     None)
        torch.cuda.synchronize()
    finally:
        del os.environ["SLP_SPLIT"]
    assert rc == 0
    want = D.decode_checksum(res, spec.kind.w, True, True)
    a = D.Substreams.from_seed(spec, 9, n)
    got = a.checksum(T, exact=True, f64=True)
    assert (got.sum, got.xor, got.mant, got.count) == (want.sum, want.xor, want.mant, want.count)
    assert abs(got.fsum_f64 - want.fsum_f64) <= 1e-12 * abs(want.fsum_f64)
    assert torch.equal(a.states, ref.states)
    b = D.Substreams.from_seed(spec, 9, n)
    out, c = D.fill_checksum(spec, b.states, T)
    assert (c.sum, c.xor, c.mant) == (want.sum, want.xor, want.mant)
    assert torch.equal(b.states, ref.states)
    d = D.Substreams.from_seed(spec, 9, n)
    assert torch.equal(out, d.fill(T))


@pytest.mark.parametrize("name,n,J", [("xoshiro256starstar", 1, 1 << 14), ("xoroshiro128plus", 3, 3000),
                                      ("xoshiro128plusplus", 40, 1500), ("xoroshiro1024starstar", 2, 1 << 12),
                                      ("xoshiro512plus", 5, 7), ("xoroshiro64star", 70000, 2)])
def test_split_substreams_segment_states(name, n, J):
    """slp_split_substreams: segment j of substream i is substream i jumped by
    j * seg steps (direct launch, radix rounds with K1 / K1t, batches of
    65535 substreams), sampled against host jumps (generators.py:315-334)."""
    import ctypes

    from paper_1805_01407_b200 import _native

    spec = P.get_spec(name)
    rng = np.random.default_rng(n * 7 + J)
    seg_len = int(rng.integers(1, 1 << 62)) << 3
    sub = D.Substreams.from_seed(spec, 21, n, stride=1 << 40)
    seg = torch.empty((spec.kind.k, n * J), dtype=sub.states.dtype, device="cuda")
    sw, sn = _native.int_to_words(seg_len)
    rc = _native.lib().slp_split_substreams(D.native_id(spec), ctypes.c_void_p(sub.states.data_ptr()), n, n, sw, sn,
                                            J, ctypes.c_void_p(seg.data_ptr()), n * J, None)
    assert rc == 0
    S = sub.states.cpu().numpy().astype(np.uint64)
    G = seg.cpu().numpy().astype(np.uint64)
    picks = {(0, 0), (n - 1, J - 1)} | {(int(rng.integers(n)), int(rng.integers(J))) for _ in range(12)}
    for i, j in sorted(picks):
        g = P.Generator.from_seed(spec, 1)
        g.set_flat_words(S[:, i])
        if j:
            g.jump(P.compute_jump_poly(spec, j * seg_len))
        assert list(g.flat_words()) == [int(v) for v in G[:, i * J + j]], (name, i, j)


def test_host_chunks_are_fresh_and_match_device_chunks():
    """Pipelined host delivery (staging double buffer + threaded copies) yields
    caller-owned arrays equal to the device chunks (generators.py:482)."""
    spec = P.get_spec("xoshiro256plusplus")
    total = 5 * 512 * 4096 + 777  # 5 full superbatches + a ragged tail
    host = list(P.LanedStream(spec, seed=9, lanes=512, lane_len=4096).chunks(total))
    dev = [c.cpu().numpy() for c in P.LanedStream(spec, seed=9, lanes=512, lane_len=4096).chunks(total, device=True)]
    assert [h.size for h in host] == [d.size for d in dev]
    for h, d in zip(host, dev):
        assert np.array_equal(h, d)
    for a in range(len(host)):
        for b in range(a + 1, len(host)):
            assert not np.shares_memory(host[a], host[b])
    host[0][:] = 0  # caller owns it: later chunks are unaffected
    assert np.array_equal(host[1], dev[1])


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro1024plusplus", "xoshiro128plusplus"])
def test_laned_fill_c_abi_superbatch(name):
    """slp_laned_fill (C ABI) = the first lanes*lane_len values of
    the scalar stream; then slp_jump_states + slp_fill give the next superbatch."""
    import ctypes

    from paper_1805_01407_b200 import _native

    spec = P.get_spec(name)
    lanes, lane_len = 96, 300
    want = O.laned_stream(name, 42, 2 * lanes * lane_len, lanes, lane_len)
    L = _native.lib()
    gid = L.slp_generator_id(name.encode())
    base = (ctypes.c_uint64 * spec.kind.k)(*O.seed_flat(name, 42))
    states = torch.empty((spec.kind.k, lanes), dtype=torch.uint64 if spec.kind.w == 64 else torch.uint32,
                         device="cuda")
    out = torch.empty((lanes, lane_len), dtype=torch.uint64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.slp_laned_fill(gid, base, lanes, lane_len, _native.OUT_U64, ctypes.c_void_p(out.data_ptr()),
                            ctypes.c_void_p(states.data_ptr()), st) == 0
    np.testing.assert_array_equal(out.cpu().numpy().reshape(-1), want[: lanes * lane_len])
    jp = P.compute_jump_poly(spec, (lanes - 1) * lane_len)
    pw, pn = _native.int_to_words(jp.poly.bits)
    sp = ctypes.c_void_p(states.data_ptr())
    assert L.slp_jump_states(gid, pw, pn, sp, lanes, sp, lanes, lanes, st) == 0
    assert L.slp_fill(gid, sp, sp, lanes, lanes, lane_len, _native.OUT_U64, _native.STREAM_MAJOR,
                      ctypes.c_void_p(out.data_ptr()), lane_len, st) == 0
    np.testing.assert_array_equal(out.cpu().numpy().reshape(-1), want[lanes * lane_len:])


@pytest.mark.parametrize("name", ["xoroshiro128plus", "xoshiro128starstar", "xoroshiro1024plusplus"])
def test_vecstepper_numpy_and_strided_states(name):
    """Drop-in use with the reference's numpy (k, L) uint64 arrays (also for
    w = 32, engines.py:276-283), and column-sliced CUDA views."""
    import random

    spec = P.get_spec(name)
    kind, params = spec.kind, spec.params
    rng = random.Random(5)
    states = [P.bits_to_words(rng.randrange(1, 1 << kind.n), kind.k, kind.w) for _ in range(7)]
    want = [tuple(s) for s in states]
    for _ in range(10):
        want = [P.step(kind, params, s) for s in want]
    # numpy uint64 host array, stepped in place
    S = np.array(list(zip(*states)), dtype=np.uint64)
    st = D.VecStepper(kind, params)
    for _ in range(10):
        st.step(S)
    assert S.dtype == np.uint64
    assert [tuple(int(v) for v in S[:, j]) for j in range(7)] == want
    S2 = np.array(list(zip(*states)), dtype=np.uint64)
    st.advance(S2, 10)
    np.testing.assert_array_equal(S2, S)
    # a column slice of a wider CUDA tensor (row pitch != L)
    npdt = np.uint64 if kind.w == 64 else np.uint32
    big = torch.zeros((kind.k, 20), dtype=torch.uint64 if kind.w == 64 else torch.uint32, device="cuda")
    big[:, 3:10] = torch.from_numpy(np.array(list(zip(*states)), dtype=npdt)).cuda()
    view = big[:, 3:10]
    for _ in range(10):
        st.step(view)
    np.testing.assert_array_equal(view.cpu().numpy().astype(np.uint64), S)
    big2 = torch.zeros_like(big)
    big2[:, 3:10] = torch.from_numpy(np.array(list(zip(*states)), dtype=npdt)).cuda()
    st.advance(big2[:, 3:10], 10)
    np.testing.assert_array_equal(big2[:, 3:10].cpu().numpy().astype(np.uint64), S)
    assert int(big2[:, :3].cpu().numpy().astype(np.uint64).sum()) == 0  # neighbours untouched


def test_fused_checksum_on_column_slice():
    """K4 on a column slice of a wider state tensor (row pitch != n) equals the
    checksum of the same substreams stored contiguously."""
    spec = P.get_spec("xoshiro512plusplus")
    sub = D.Substreams.from_seed(spec, 42, 300)
    ref = sub.states[:, 100:250].clone()
    c_ref = D.fused_checksum(spec, ref, 333)
    view = sub.states[:, 100:250]
    c_view = D.fused_checksum(spec, view, 333)
    assert (c_view.sum, c_view.xor, c_view.mant) == (c_ref.sum, c_ref.xor, c_ref.mant)
    assert torch.equal(view, ref)  # advanced in place, identically
    assert torch.equal(sub.states[:, :100], D.Substreams.from_seed(spec, 42, 300).states[:, :100])


def test_host_chunks_sliced_staging(monkeypatch):
    """A superbatch larger than the pinned staging slice is delivered through
    several slices (bounded pinned memory), unchanged."""
    monkeypatch.setattr(P.LanedStream, "_STAGE_VALUES", 1000)
    spec = P.get_spec("xoroshiro128plusplus")
    total = 3 * 64 * 500 + 123
    host = list(P.LanedStream(spec, seed=4, lanes=64, lane_len=500).chunks(total))
    want = O.laned_stream("xoroshiro128plusplus", 4, total, 64, 500)
    np.testing.assert_array_equal(np.concatenate(host), want)
    assert [h.size for h in host] == [32000, 32000, 32000, 123]
    views = [v.copy() for v in P.LanedStream(spec, seed=4, lanes=64, lane_len=500).chunks(total, _views=True)]
    np.testing.assert_array_equal(np.concatenate(views), want)

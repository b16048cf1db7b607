"""Pin the CPU oracle (oracle/oracle.py) to the reference's golden vectors
(tests/golden/*.json, produced by tests/golden/make_golden.py from the
reference itself).  CPU only."""

import numpy as np
import pytest

from oracle import oracle as O

NAMES = O.REGISTRY_NAMES


def hexs(vals):
    return [hex(int(v)) for v in vals]


def test_splitmix_kats(G):
    kat = G("splitmix64")
    assert hexs(O.splitmix64(0, 8)) == kat["splitmix64_seed0"]
    assert hexs(O.splitmix64(42, 8)) == kat["splitmix64_seed42"]
    # test_generators.py:72-76
    assert O.splitmix64(0, 2) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]


@pytest.mark.parametrize("name", NAMES)
def test_seed_states(G, name):
    d = G("generators")[name]
    for seed, want in d["seed_states"].items():
        assert hexs(O.seed_state(name, int(seed))) == want


@pytest.mark.parametrize("name", NAMES)
def test_outputs_and_states(G, name):
    d = G("generators")[name]
    for seed in (42, 7):
        outs, st = O.outputs(name, O.seed_flat(name, seed), 100)
        assert hexs(outs) == d[f"first_outputs_seed{seed}"]
        assert hexs(st) == d[f"state_after_100_seed{seed}"]
    if O.SPECS[name][2] == 64:
        outs, _ = O.outputs(name, O.seed_flat(name, 42), 16)
        assert [float.hex(float(x)) for x in O.to_f64(outs)] == d["first_doubles_seed42"]


@pytest.mark.parametrize("name", NAMES)
def test_jumps(G, name):
    d = G("generators")[name]
    e = G("engines")[O.engine_key(name)]
    n = O.SPECS[name][1] * O.SPECS[name][2]
    jp = O.jump_poly(name, 1 << (n // 2))
    assert hex(jp) == e["jump_poly"]
    st = O.jump(name, O.seed_flat(name, 42), jp)
    assert hexs(st) == d["jump_state_seed42"]
    outs, _ = O.outputs(name, st, 32)
    assert hexs(outs) == d["jump_outputs_seed42"][:32]
    if n <= 256:
        lj = O.jump_poly(name, 1 << (3 * n // 4))
        assert hex(lj) == e["long_jump_poly"]
        assert hexs(O.jump(name, O.seed_flat(name, 42), lj)) == d["long_jump_state_seed42"]
    assert hex(O.jump_poly(name, 12345)) == e["x_pow_12345"]


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoroshiro128plus", "xoshiro128starstar",
                                  "xoroshiro64star", "xoroshiro128plusplus"])
def test_lane_states_dense(G, name):
    d = G("substreams")[name]
    n = O.SPECS[name][1] * O.SPECS[name][2]
    S = O.lane_states(name, O.seed_flat(name, d["seed"]), 64, 1 << (n // 2))
    for i in range(64):
        assert hexs(S[:, i]) == d["dense_states"][i]


@pytest.mark.parametrize("key", ["xoroshiro128plus/5/2500/6/128", "xoshiro256plus/8/700/1/256",
                                 "xoroshiro64starstar/3/3000/5/256", "xorshift128/5/2500/6/128"])
def test_laned_stream(G, key):
    d = G("laned")[key]
    vals = O.laned_stream(d["name"], d["seed"], d["total"], d["lanes"], d["lane_len"])
    assert hexs(vals) == d["values"]


@pytest.mark.parametrize("key", ["c2s/xoshiro256starstar", "c3s/xoroshiro128plusplus", "c4s/xoroshiro64starstar"])
def test_small_checksums(G, key):
    g = G("checksums_small")[key]
    name = g["name"]
    n = O.SPECS[name][1] * O.SPECS[name][2]
    S = O.lane_states(name, O.seed_flat(name, g["seed"]), g["substreams"], 1 << (n // 2))
    outs, _ = O.vec_outputs(name, S, g["T"])
    c = O.checksum(outs, O.SPECS[name][2])
    assert hex(c["sum"]) == g["sum"] and hex(c["xor"]) == g["xor"] and hex(c["mant"]) == g["mant"]


def test_f32_conversion_exact():
    x = np.array([0, 0xFF, 0x100, 0xFFFFFFFF, 0x80000000, 0x12345678], dtype=np.uint64)
    f = O.to_f32(x)
    assert f[0] == 0.0 and f[1] == 0.0 and f[2] == 2.0 ** -24
    assert f[3] == np.float32((2 ** 24 - 1) / 2 ** 24) and f[4] == 0.5
    assert float(f[5]) == (0x12345678 >> 8) / 2 ** 24

"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy / Python-int restatement of the reference algorithm for the hot path
(the `slprng` package, /root/reference/pkg/src/slprng/).  Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may import it,
and only as the checker; the product (paper_1805_01407_b200) never does.

Parity is PINNED: tests/test_oracle.py checks every function below against
the golden vectors in tests/golden/, which tests/golden/make_golden.py
produced by running the reference itself.  The characteristic polynomials
are taken from that golden data (tests/golden/engines.json, the reference's
own ``engine_char_poly`` output), not recomputed.

Each function cites the reference lines it restates.
"""

from __future__ import annotations

import json
import os

import numpy as np

M64 = (1 << 64) - 1
_GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

# name -> (family, k, w, (a, b, c), scrambler, i, j, S, R, T)        generators.py:71-110
SPECS = {
    "xoroshiro128": ("xoroshiro", 2, 64, (24, 16, 37), "none", 0, None, None, None, None),
    "xoroshiro128plus": ("xoroshiro", 2, 64, (24, 16, 37), "plus", 0, 1, None, None, None),
    "xoroshiro128star": ("xoroshiro", 2, 64, (24, 16, 37), "star", 0, None, 0x9E3779B97F4A7C13, None, None),
    "xoroshiro128plusplus": ("xoroshiro", 2, 64, (49, 21, 28), "plusplus", 0, 1, None, 17, None),
    "xoroshiro128starstar": ("xoroshiro", 2, 64, (24, 16, 37), "starstar", 0, None, 5, 7, 9),
    "xoshiro256": ("xoshiro", 4, 64, (17, 45, None), "none", 1, None, None, None, None),
    "xoshiro256plus": ("xoshiro", 4, 64, (17, 45, None), "plus", 0, 3, None, None, None),
    "xoshiro256plusplus": ("xoshiro", 4, 64, (17, 45, None), "plusplus", 0, 3, None, 23, None),
    "xoshiro256starstar": ("xoshiro", 4, 64, (17, 45, None), "starstar", 1, None, 5, 7, 9),
    "xoshiro512": ("xoshiro", 8, 64, (11, 21, None), "none", 1, None, None, None, None),
    "xoshiro512plus": ("xoshiro", 8, 64, (11, 21, None), "plus", 0, 2, None, None, None),
    "xoshiro512plusplus": ("xoshiro", 8, 64, (11, 21, None), "plusplus", 2, 0, None, 17, None),
    "xoshiro512starstar": ("xoshiro", 8, 64, (11, 21, None), "starstar", 1, None, 5, 7, 9),
    "xoroshiro1024": ("xoroshiro", 16, 64, (25, 27, 36), "none", 0, None, None, None, None),
    "xoroshiro1024plus": ("xoroshiro", 16, 64, (25, 27, 36), "plus", 0, 15, None, None, None),
    "xoroshiro1024star": ("xoroshiro", 16, 64, (25, 27, 36), "star", 0, None, 0x9E3779B97F4A7C13, None, None),
    "xoroshiro1024plusplus": ("xoroshiro", 16, 64, (25, 27, 36), "plusplus", 15, 0, None, 23, None),
    "xoroshiro1024starstar": ("xoroshiro", 16, 64, (25, 27, 36), "starstar", 0, None, 5, 7, 9),
    "xoroshiro64": ("xoroshiro", 2, 32, (26, 9, 13), "none", 0, None, None, None, None),
    "xoroshiro64star": ("xoroshiro", 2, 32, (26, 9, 13), "star", 0, None, 0x9E3779BB, None, None),
    "xoroshiro64starstar": ("xoroshiro", 2, 32, (26, 9, 13), "starstar", 0, None, 0x9E3779BB, 5, 5),
    "xoshiro128": ("xoshiro", 4, 32, (9, 11, None), "none", 1, None, None, None, None),
    "xoshiro128plus": ("xoshiro", 4, 32, (9, 11, None), "plus", 0, 3, None, None, None),
    "xoshiro128plusplus": ("xoshiro", 4, 32, (9, 11, None), "plusplus", 0, 3, None, 7, None),
    "xoshiro128starstar": ("xoshiro", 4, 32, (9, 11, None), "starstar", 1, None, 5, 7, 9),
    "xorshift128": ("xorshift", 2, 64, (23, 17, 26), "none", 0, None, None, None, None),
    "xorshift128plus": ("xorshift", 2, 64, (23, 17, 26), "plus", 0, 1, None, None, None),
}


REGISTRY_NAMES = list(SPECS)  # the reference registry; custom engines are appended below


def _load_custom():
    """Engines built with the reference's custom_spec (generators.py:127-135):
    specs and char polys from tests/golden/custom.json (make_golden_custom.py,
    produced by the reference)."""
    path = os.path.join(_GOLDEN, "custom.json")
    if not os.path.exists(path):
        return {}
    with open(path) as f:
        data = json.load(f)
    polys = {}
    for name, d in data.items():
        sc = d["scrambler"]
        SPECS[name] = (d["family"], d["k"], d["w"], (d["a"], d["b"], d["c"]), sc["kind"], sc.get("word_i", 0),
                       sc.get("word_j"), sc.get("S"), sc.get("R"), sc.get("T"))
        polys[f"{d['family']}-{d['k']}-{d['w']}-{d['a']}-{d['b']}-{d['c']}"] = int(d["char_poly"], 16)
    return polys


_CUSTOM_POLYS = _load_custom()


def engine_key(name):
    fam, k, w, (a, b, c), *_ = SPECS[name]
    return f"{fam}-{k}-{w}-{a}-{b}-{c}"


# ---------------------------------------------------------------- seeding


def splitmix64(seed: int, count: int):
    """generators.py:142-150"""
    x = seed & M64
    out = []
    for _ in range(count):
        x = (x + 0x9E3779B97F4A7C15) & M64
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        out.append(z ^ (z >> 31))
    return out


def seed_state(name: str, seed: int):
    """generators.py:153-181 (w = 64 / 32)"""
    _, k, w, *_ = SPECS[name]
    if w == 64:
        return splitmix64(seed, k)
    words = []
    for z in splitmix64(seed, (k + 1) // 2):
        words += [z & 0xFFFFFFFF, z >> 32]
    return words[:k]


def seed_flat(name: str, seed: int):
    """Flat view of Generator.from_seed (generators.py:217-219, 226-232): the
    ring engines (xoroshiro, k > 2) start with pointer 0, so flat word i is
    storage word (1 + i) mod k."""
    fam, k, *_ = SPECS[name]
    words = seed_state(name, seed)
    if fam == "xoroshiro" and k > 2:
        return [words[(1 + i) % k] for i in range(k)]
    return words


# ---------------------------------------------------------------- scalar


def _rotl(x, r, w):
    m = (1 << w) - 1
    return ((x << r) | (x >> (w - r))) & m


def step(name, s):
    """engines.py:100-140, flat view"""
    fam, k, w, (a, b, c), *_ = SPECS[name]
    m = (1 << w) - 1
    s = list(s)
    if fam == "xoroshiro":
        x0 = s[0]
        xl = s[-1] ^ x0
        return s[1:k - 1] + [_rotl(x0, a, w) ^ xl ^ ((xl << b) & m), _rotl(xl, c, w)]
    if fam == "xorshift":
        t = s[0] ^ ((s[0] << a) & m)
        return [s[1], t ^ (t >> b) ^ s[1] ^ (s[1] >> c)]
    t = (s[1] << a) & m
    if k == 4:
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t  # noqa: E702
        s[3] = _rotl(s[3], b, w)
    else:
        s[2] ^= s[0]; s[5] ^= s[1]; s[1] ^= s[2]; s[7] ^= s[3]; s[3] ^= s[4]  # noqa: E702
        s[4] ^= s[5]; s[0] ^= s[6]; s[6] ^= s[7]; s[6] ^= t  # noqa: E702
        s[7] = _rotl(s[7], b, w)
    return s


def scramble(name, s):
    """scramblers.py:84-95"""
    _, k, w, _, kind, i, j, S, R, T = SPECS[name]
    m = (1 << w) - 1
    x = s[i]
    if kind == "none":
        return x
    if kind == "plus":
        return (x + s[j]) & m
    if kind == "star":
        return (x * S) & m
    if kind == "plusplus":
        return (_rotl((x + s[j]) & m, R, w) + x) & m
    return (_rotl((x * S) & m, R, w) * T) & m


def outputs(name, flat, count):
    """generators.py:244-305 in the flat view: scramble, then step."""
    s = list(flat)
    out = []
    for _ in range(count):
        out.append(scramble(name, s))
        s = step(name, s)
    return out, s


# ---------------------------------------------------------------- GF(2) / jumps


_golden_engines = None


def char_poly(name) -> int:
    """The reference's own engine_char_poly output (tests/golden/engines.json)."""
    global _golden_engines
    if _golden_engines is None:
        with open(os.path.join(_GOLDEN, "engines.json")) as f:
            _golden_engines = json.load(f)
    key = engine_key(name)
    if key in _golden_engines:
        return int(_golden_engines[key]["char_poly"], 16)
    return _CUSTOM_POLYS[key]


def _clmul(a, b):
    r = 0
    while a:
        low = a & -a
        r ^= b << (low.bit_length() - 1)
        a ^= low
    return r


def _mod(a, m):
    dm = m.bit_length() - 1
    while a.bit_length() - 1 >= dm:
        a ^= m << (a.bit_length() - 1 - dm)
    return a


def x_pow_mod(e: int, P: int) -> int:
    """gf2.py:214-227: x**e mod P by square-and-multiply"""
    r, b = 1, _mod(2, P)
    while e:
        if e & 1:
            r = _mod(_clmul(r, b), P)
        e >>= 1
        if e:
            b = _mod(_clmul(b, b), P)
    return r


def jump_poly(name, steps: int) -> int:
    """generators.py:397-402"""
    return x_pow_mod(steps, char_poly(name))


def jump(name, flat, poly_bits):
    """generators.py:315-334"""
    cur = list(flat)
    acc = [0] * len(cur)
    deg = poly_bits.bit_length() - 1
    for d in range(deg + 1):
        if (poly_bits >> d) & 1:
            acc = [x ^ y for x, y in zip(acc, cur)]
        if d != deg:
            cur = step(name, cur)
    return acc


# ---------------------------------------------------------------- vectorised lanes


def vec_step(name, S):
    """engines.py:318-361 on a (k, L) uint64 array (rows physically rolled for ring engines)."""
    fam, k, w, (a, b, c), *_ = SPECS[name]
    m = np.uint64((1 << w) - 1)

    def rl(x, r):
        return ((x << np.uint64(r)) | (x >> np.uint64(w - r))) & m

    if fam == "xoroshiro":
        x0 = S[0]
        xl = S[k - 1] ^ x0
        new = np.empty_like(S)
        new[: k - 2] = S[1: k - 1]
        new[k - 2] = rl(x0, a) ^ xl ^ ((xl << np.uint64(b)) & m)
        new[k - 1] = rl(xl, c)
        return new
    if fam == "xorshift":
        t = S[0] ^ ((S[0] << np.uint64(a)) & m)
        return np.stack([S[1], t ^ (t >> np.uint64(b)) ^ S[1] ^ (S[1] >> np.uint64(c))])
    S = S.copy()
    t = (S[1] << np.uint64(a)) & m
    if k == 4:
        S[2] ^= S[0]; S[3] ^= S[1]; S[1] ^= S[2]; S[0] ^= S[3]; S[2] ^= t  # noqa: E702
        S[3] = rl(S[3], b)
    else:
        S[2] ^= S[0]; S[5] ^= S[1]; S[1] ^= S[2]; S[7] ^= S[3]; S[3] ^= S[4]  # noqa: E702
        S[4] ^= S[5]; S[0] ^= S[6]; S[6] ^= S[7]; S[6] ^= t  # noqa: E702
        S[7] = rl(S[7], b)
    return S


def vec_scramble(name, S):
    """scramblers.py:97-127"""
    _, k, w, _, kind, i, j, Sm, R, T = SPECS[name]
    m = np.uint64((1 << w) - 1)
    x = S[i]
    with np.errstate(over="ignore"):
        if kind == "none":
            return x.copy()
        if kind == "plus":
            return (x + S[j]) & m
        if kind == "star":
            return (x * np.uint64(Sm)) & m
        r, wr = np.uint64(R), np.uint64(w - R)
        if kind == "plusplus":
            t = (x + S[j]) & m
            return ((((t << r) | (t >> wr)) & m) + x) & m
        z = (x * np.uint64(Sm)) & m
        return ((((z << r) | (z >> wr)) & m) * np.uint64(T)) & m


def vec_outputs(name, S, T):
    """T outputs of each lane of the flat (k, L) states: returns ((L, T) uint64, new states)."""
    S = np.asarray(S, dtype=np.uint64)
    buf = np.empty((T, S.shape[1]), dtype=np.uint64)
    for t in range(T):
        buf[t] = vec_scramble(name, S)
        S = vec_step(name, S)
    return buf.T.copy(), S


def vec_jump(name, S, poly_bits):
    """generators.py:493-505"""
    cur = np.asarray(S, dtype=np.uint64).copy()
    acc = np.zeros_like(cur)
    deg = poly_bits.bit_length() - 1
    for d in range(deg + 1):
        if (poly_bits >> d) & 1:
            acc ^= cur
        if d != deg:
            cur = vec_step(name, cur)
    return acc


def lane_states(name, flat0, lanes, lane_len):
    """generators.py:443-459: lane j = flat0 jumped j*lane_len, by doubling."""
    _, k, *_ = SPECS[name]
    S = np.zeros((k, lanes), dtype=np.uint64)
    S[:, 0] = np.array(flat0, dtype=np.uint64)
    if lanes > 1:
        P = char_poly(name)
        g = x_pow_mod(lane_len, P)
        filled = 1
        while filled < lanes:
            mm = min(filled, lanes - filled)
            S[:, filled: filled + mm] = vec_jump(name, S[:, :mm], g)
            g = _mod(_clmul(g, g), P)
            filled += mm
    return S


def laned_stream(name, seed, total, lanes, lane_len):
    """generators.py:426-513 (output_stream with the lanes clamp); returns the concatenation."""
    lanes = max(1, min(lanes, -(-total // lane_len)))
    S = lane_states(name, seed_flat(name, seed), lanes, lane_len)
    sj = jump_poly(name, (lanes - 1) * lane_len) if lanes > 1 else None
    parts, produced = [], 0
    while produced < total:
        out, S = vec_outputs(name, S, lane_len)
        chunk = out.reshape(-1)[: total - produced]
        parts.append(chunk)
        produced += chunk.size
        if sj is not None:
            S = vec_jump(name, S, sj)
    return np.concatenate(parts)


def checksum(values: np.ndarray, w: int):
    """sum mod 2^64, xor, exact sum of x >> (11|8) over an array of outputs."""
    v = np.asarray(values, dtype=np.uint64).reshape(-1)
    shift = 11 if w == 64 else 8
    hi = (v >> np.uint64(32)).astype(object).sum() if v.size else 0
    lo = (v & np.uint64(0xFFFFFFFF)).astype(object).sum() if v.size else 0
    exact = (int(hi) << 32) + int(lo)
    m = v >> np.uint64(shift)
    mant = (int((m >> np.uint64(32)).astype(object).sum()) << 32) + int((m & np.uint64(0xFFFFFFFF)).astype(object).sum()) \
        if v.size else 0
    x = int(np.bitwise_xor.reduce(v)) if v.size else 0
    return {"sum": exact & M64, "xor": x, "mant": mant}


def to_f64(values):
    """generators.py:307-311 elementwise: (x >> 11) * 2^-53"""
    return (np.asarray(values, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def to_f32(values):
    """north_star u32 -> float: (x >> 8) * 2^-24 (no reference function; exact)"""
    return ((np.asarray(values, dtype=np.uint64) >> np.uint64(8)).astype(np.float32) * np.float32(2.0 ** -24))


def hwd_test_values(name, seed, n_values, split=False, transitional=False, w_test=64):
    """The first n_values HWD test values of a generator's stream:
    hwd.py:473-476 split (low half first) then :446-470 transitional (carry 0)."""
    factor = 2 if split else 1
    src = laned_stream(name, seed, -(-n_values // factor), 64, 4096)
    if split:
        v = src.astype(np.uint64).view(np.uint32).astype(np.uint64)[:n_values]
    else:
        v = src[:n_values].astype(np.uint64)
    if transitional:
        m = np.uint64((1 << w_test) - 1) if w_test < 64 else None
        prev = np.concatenate([np.zeros(1, np.uint64), v[:-1]])
        sh = (v << np.uint64(1)) | (prev >> np.uint64(w_test - 1))
        if m is not None:
            sh &= m
        v = v ^ sh
    return v


def hwd_counts(values, c0, c1, k, w_test, ell):
    """Per-signature counts and weight sums of positions [c0, c1) of a test-value
    array (hwd.py:206-233 HwdCounters._add, signatures from the k previous trits)."""
    v = np.asarray(values, dtype=np.uint64)
    nu = np.bitwise_count(v).astype(np.int64)
    lo, hi = w_test // 2 - ell, w_test // 2 + ell
    trits = (nu >= lo).astype(np.int64) + (nu > hi)
    pos = np.arange(c0, c1)
    sig = np.zeros(pos.size, dtype=np.int64)
    for j in range(1, k + 1):
        sig += trits[pos - j] * 3 ** (k - j)
    counts = np.bincount(sig, minlength=3 ** k).astype(np.uint64)
    sums = np.bincount(sig, weights=nu[pos].astype(np.float64), minlength=3 ** k).astype(np.uint64)
    return counts, sums

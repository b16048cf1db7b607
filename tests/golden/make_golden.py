"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
itself (the `slprng` package at /root/reference/pkg/src, imported read-only).

This script is test infrastructure: it runs only in the build container, where
/root/reference exists.  Its outputs (small JSON files) are committed so that
the GPU box, which has no /root/reference, can check against them.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py            # small fixtures
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py --big      # + full-size config checksums

Everything is produced through the reference's public functions only:
`Generator.from_seed/next/next_double/jump` (generators.py:188-334),
`seed_state`/`splitmix64` (:142-181), `engine_char_poly`/`compute_jump_poly`/
`default_jumps` (:387-419), `LanedStream`/`output_stream` (:426-513),
`VecStepper` (engines.py:276-361) and `ScramblerSpec.apply_vec`
(scramblers.py:97-127).  The config checksums follow the recipe of SURVEY.md
Appendix A (per-task jump to (b << 3n/4) + (c0 << n/2), LanedStream lanes,
T x (apply_vec, step)).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402
from slprng import generators  # noqa: E402
from slprng.engines import VecStepper  # noqa: E402
from slprng.generators import (  # noqa: E402
    Generator,
    LanedStream,
    compute_jump_poly,
    default_jumps,
    engine_char_poly,
    get_spec,
    output_stream,
    registry_names,
    seed_state,
    splitmix64,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def hx(v: int) -> str:
    return f"0x{v:x}"


def hexlist(vs):
    return [hx(int(v)) for v in vs]


# ---------------------------------------------------------------------------
# small fixtures


def engine_fixtures():
    """Char polys and default jump polys per engine_key."""
    out = {}
    for name in registry_names(include_analysis=True):
        spec = get_spec(name)
        key = spec.engine_key
        skey = "-".join(str(x) for x in key)
        if skey in out:
            out[skey]["generators"].append(name)
            continue
        t0 = time.time()
        P = engine_char_poly(spec)
        j, lj = default_jumps(spec)
        out[skey] = {
            "family": spec.kind.family, "k": spec.kind.k, "w": spec.kind.w,
            "a": spec.params.a, "b": spec.params.b, "c": spec.params.c,
            "char_poly": hx(P.bits),
            "jump_steps": hx(j.step_count), "jump_poly": hx(j.poly.bits),
            "long_jump_steps": hx(lj.step_count), "long_jump_poly": hx(lj.poly.bits),
            # a few extra powers used by the device doubling init
            "x_pow_1024": hx(compute_jump_poly(spec, 1024).poly.bits),
            "x_pow_4096": hx(compute_jump_poly(spec, 4096).poly.bits),
            "x_pow_12345": hx(compute_jump_poly(spec, 12345).poly.bits),
            "generators": [name],
        }
        print(f"  engine {skey}: {time.time() - t0:.1f}s", flush=True)
    return out


def generator_fixtures():
    out = {}
    for name in registry_names(include_analysis=True):
        spec = get_spec(name)
        w = spec.kind.w
        d = {"w": w, "k": spec.kind.k, "seed_states": {}}
        for seed in (0, 1, 7, 42, 2024, (1 << 64) - 1):
            d["seed_states"][str(seed)] = hexlist(seed_state(spec, seed))
        for seed in (42, 7):
            g = Generator.from_seed(spec, seed)
            d[f"first_outputs_seed{seed}"] = hexlist(g.next() for _ in range(100))
            d[f"state_after_100_seed{seed}"] = hexlist(g.flat_words())
        if w == 64:
            g = Generator.from_seed(spec, 42)
            d["first_doubles_seed42"] = [float.hex(g.next_double()) for _ in range(16)]
        j, lj = default_jumps(spec)
        g = Generator.from_seed(spec, 42).jump(j)
        d["jump_state_seed42"] = hexlist(g.flat_words())
        d["jump_outputs_seed42"] = hexlist(g.next() for _ in range(1024 if name == "xoshiro256starstar" else 32))
        g = Generator.from_seed(spec, 42).jump(lj)
        d["long_jump_state_seed42"] = hexlist(g.flat_words())
        d["long_jump_outputs_seed42"] = hexlist(g.next() for _ in range(32))
        out[name] = d
    return out


def substream_fixtures():
    """Substream states stream i = seed state jumped i * 2^(n/2) (configs 2-5),
    obtained from the reference's own LanedStream doubling (generators.py:450-459)
    and, for sparse indices, from compute_jump_poly + Generator.jump."""
    out = {}
    cases = [
        ("xoshiro256starstar", 42), ("xoroshiro128plus", 42), ("xoroshiro128plusplus", 42),
        ("xoshiro512starstar", 42), ("xoroshiro1024starstar", 42),
        ("xoshiro128starstar", 7), ("xoroshiro64star", 7),
    ]
    for name, seed in cases:
        spec = get_spec(name)
        n = spec.kind.n
        J = 1 << (n // 2)
        lanes = 64
        g = Generator.from_seed(spec, seed)
        S = LanedStream(spec, generator=g, lanes=lanes, lane_len=J).S
        dense = [hexlist(S[:, i]) for i in range(lanes)]
        sparse = {}
        for i in (1023, 4097, (1 << 20) - 1, (1 << 22) - 1):
            h = Generator.from_seed(spec, seed).jump(compute_jump_poly(spec, i * J))
            sparse[str(i)] = hexlist(h.flat_words())
        # long-jump blocks (config 5 decomposition): block b base state
        blocks = {}
        for b in range(1, 8):
            h = Generator.from_seed(spec, seed).jump(compute_jump_poly(spec, b << (3 * n // 4)))
            blocks[str(b)] = hexlist(h.flat_words())
        out[name] = {"seed": seed, "J_log2": n // 2, "dense_states": dense,
                     "sparse_states": sparse, "long_jump_blocks": blocks}
    return out


def laned_fixtures():
    """output_stream / LanedStream.chunks parity cases (test_generators.py:213-231)."""
    out = {}
    cases = [
        ("xoroshiro128plus", 5, 2500, 6, 128), ("xoshiro256starstar", 5, 2500, 6, 128),
        ("xoroshiro1024plusplus", 5, 2500, 6, 128), ("xorshift128", 5, 2500, 6, 128),
        ("xoshiro128plus", 5, 2500, 6, 128), ("xoshiro256plus", 8, 700, 1, 256),
        ("xoshiro256starstar", 42, 5000, 4, 1000), ("xoroshiro64starstar", 3, 3000, 5, 256),
        ("xoshiro512plusplus", 11, 4096, 8, 128),
    ]
    for name, seed, total, lanes, lane_len in cases:
        spec = get_spec(name)
        chunks = list(output_stream(spec, seed=seed, total_values=total, lanes=lanes, lane_len=lane_len))
        vals = np.concatenate(chunks)
        out[f"{name}/{seed}/{total}/{lanes}/{lane_len}"] = {
            "name": name, "seed": seed, "total": total, "lanes": lanes, "lane_len": lane_len,
            "chunk_sizes": [int(c.size) for c in chunks],
            "values": hexlist(vals),
        }
    return out


# ---------------------------------------------------------------------------
# checksums over (block, substream, position): SURVEY.md Appendix A recipe


def _task(args):
    name, seed, b, c0, c1, T = args
    spec = get_spec(name)
    n, w = spec.kind.n, spec.kind.w
    g = Generator.from_seed(spec, seed)
    off = (b << (3 * n // 4)) + (c0 << (n // 2))
    if off:
        g.jump(compute_jump_poly(spec, off))
    lanes = c1 - c0
    S = LanedStream(spec, generator=g, lanes=lanes, lane_len=1 << (n // 2)).S
    st = VecStepper(spec.kind, spec.params)
    sc = spec.scrambler
    shift = np.uint64(11 if w == 64 else 8)
    s_sum = np.zeros(lanes, dtype=np.uint64)
    s_xor = np.zeros(lanes, dtype=np.uint64)
    mant_total = 0
    m_acc = np.zeros(lanes, dtype=np.uint64)
    for t in range(T):
        xi = st.word(S, sc.word_i)
        xj = st.word(S, sc.word_j) if sc.word_j is not None else None
        v = sc.apply_vec(xi, xj, w)
        s_sum += v
        s_xor ^= v
        m_acc += v >> shift
        if (t & 511) == 511:  # (x>>11) < 2^53: 512 of them fit in uint64
            mant_total += int((m_acc >> np.uint64(32)).sum()) << 32
            mant_total += int((m_acc & np.uint64(0xFFFFFFFF)).sum())
            m_acc[:] = 0
        st.step(S)
    mant_total += int((m_acc >> np.uint64(32)).sum()) << 32
    mant_total += int((m_acc & np.uint64(0xFFFFFFFF)).sum())
    tot = int((s_sum >> np.uint64(32)).sum()) << 32
    tot += int((s_sum & np.uint64(0xFFFFFFFF)).sum())
    x = int(np.bitwise_xor.reduce(s_xor)) if lanes else 0
    return tot, x, mant_total


def checksum(name, seed, blocks, S, T, procs, chunk=1 << 13):
    tasks = []
    for b in range(blocks):
        for c0 in range(0, S, chunk):
            tasks.append((name, seed, b, c0, min(S, c0 + chunk), T))
    if procs > 1:
        with mp.Pool(procs) as pool:
            res = pool.map(_task, tasks, chunksize=1)
    else:
        res = [_task(t) for t in tasks]
    tot = sum(r[0] for r in res)
    x = 0
    for r in res:
        x ^= r[1]
    mant = sum(r[2] for r in res)
    w = get_spec(name).kind.w
    scale = 53 if w == 64 else 24
    import fractions
    fsum = float(fractions.Fraction(mant, 1 << scale))
    return {"sum": hx(tot & ((1 << 64) - 1)), "xor": hx(x), "mant": hx(mant),
            "fsum": float.hex(fsum)}


SMALL_CHECKSUMS = [
    # (config, name, seed, blocks, S, T)
    ("c2s", "xoshiro256plus", 42, 1, 4096, 1024),
    ("c2s", "xoshiro256plusplus", 42, 1, 4096, 1024),
    ("c2s", "xoshiro256starstar", 42, 1, 4096, 1024),
    ("c3s", "xoroshiro128plus", 42, 1, 4096, 1024),
    ("c3s", "xoroshiro128plusplus", 42, 1, 4096, 1024),
    ("c3s", "xoroshiro128starstar", 42, 1, 4096, 1024),
    ("c4s", "xoshiro128starstar", 7, 1, 4096, 1024),
    ("c4s", "xoshiro128plusplus", 7, 1, 4096, 1024),
    ("c4s", "xoroshiro64star", 7, 1, 4096, 1024),
    ("c4s", "xoroshiro64starstar", 7, 1, 4096, 1024),
    ("c5s", "xoshiro512starstar", 42, 8, 256, 2048),
    ("c5s", "xoshiro512plusplus", 42, 8, 256, 2048),
    ("c5s", "xoroshiro1024starstar", 42, 8, 256, 2048),
    ("c5s", "xoroshiro1024plusplus", 42, 8, 256, 2048),
]

BIG_CHECKSUMS = [
    ("c2", "xoshiro256plus", 42, 1, 1 << 20, 1024),
    ("c2", "xoshiro256plusplus", 42, 1, 1 << 20, 1024),
    ("c2", "xoshiro256starstar", 42, 1, 1 << 20, 1024),
    ("c3", "xoroshiro128plus", 42, 1, 1 << 21, 1024),
    ("c3", "xoroshiro128plusplus", 42, 1, 1 << 21, 1024),
    ("c3", "xoroshiro128starstar", 42, 1, 1 << 21, 1024),
    ("c4", "xoshiro128starstar", 7, 1, 1 << 22, 1024),
    ("c4", "xoshiro128plusplus", 7, 1, 1 << 22, 1024),
    ("c4", "xoroshiro64star", 7, 1, 1 << 22, 1024),
    ("c4", "xoroshiro64starstar", 7, 1, 1 << 22, 1024),
    ("c5", "xoshiro512starstar", 42, 8, 1 << 18, 1 << 13),
    ("c5", "xoshiro512plusplus", 42, 8, 1 << 18, 1 << 13),
    ("c5", "xoroshiro1024starstar", 42, 8, 1 << 18, 1 << 13),
    ("c5", "xoroshiro1024plusplus", 42, 8, 1 << 18, 1 << 13),
]


def run_checksums(cases, procs, path):
    res = {}
    if os.path.exists(path):
        with open(path) as f:
            res = json.load(f)
    for cfg, name, seed, blocks, S, T in cases:
        key = f"{cfg}/{name}"
        if key in res:
            continue
        t0 = time.time()
        r = checksum(name, seed, blocks, S, T, procs)
        r.update({"config": cfg, "name": name, "seed": seed, "blocks": blocks,
                  "substreams": S, "T": T, "ref_seconds": round(time.time() - t0, 1), "procs": procs})
        res[key] = r
        print(f"  {key}: {r['sum']} {r['xor']} ({r['ref_seconds']}s)", flush=True)
        with open(path, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also full-size config checksums (minutes)")
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--only", default=None, help="comma list of parts: engines,generators,substreams,laned,small,big")
    args = ap.parse_args()
    parts = set((args.only or "engines,generators,substreams,laned,small").split(","))
    if args.big:
        parts.add("big")

    def dump(obj, fname):
        with open(os.path.join(HERE, fname), "w") as f:
            json.dump(obj, f, indent=1, sort_keys=True)

    kat = {"splitmix64_seed0": [hx(v) for v, _ in zip(splitmix64(0), range(8))],
           "splitmix64_seed42": [hx(v) for v, _ in zip(splitmix64(42), range(8))]}
    dump(kat, "splitmix64.json")
    if "engines" in parts:
        print("engines", flush=True)
        dump(engine_fixtures(), "engines.json")
    if "generators" in parts:
        print("generators", flush=True)
        dump(generator_fixtures(), "generators.json")
    if "substreams" in parts:
        print("substreams", flush=True)
        dump(substream_fixtures(), "substreams.json")
    if "laned" in parts:
        print("laned", flush=True)
        dump(laned_fixtures(), "laned.json")
    if "small" in parts:
        print("small checksums", flush=True)
        run_checksums(SMALL_CHECKSUMS, args.procs, os.path.join(HERE, "checksums_small.json"))
    if "big" in parts:
        print("big checksums", flush=True)
        run_checksums(BIG_CHECKSUMS, args.procs, os.path.join(HERE, "checksums_big.json"))


if __name__ == "__main__":
    main()

"""Golden fixtures for engines built with the reference's ``custom_spec``
(generators.py:127-135): tests/golden/custom.json, produced by running the
REFERENCE itself (imported read-only from /root/reference/pkg/src; test
infrastructure, build container only).

One entry per custom generator, covering every engine shape the device's
run-time parameter kernels serve plus one shape they do not:
  * the reference's ``engine_char_poly`` and jump polynomial x^(2^(n/2));
  * the first 100 outputs of ``Generator.from_seed(spec, 42)``;
  * 40 substream states ``LanedStream(spec, seed=42, lanes=40,
    lane_len=2^(n/2)).S`` (flat words, generators.py:435-463);
  * ``output_stream(spec, 42, 3000, lanes=5, lane_len=512)`` (:508-513);
  * the same 40 states after 64 ``VecStepper.step`` calls (engines.py:318-361).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_custom.py
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from slprng.engines import VecStepper  # noqa: E402
from slprng.generators import (  # noqa: E402
    Generator,
    LanedStream,
    compute_jump_poly,
    custom_spec,
    engine_char_poly,
    output_stream,
)
from slprng.scramblers import ScramblerSpec  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, family, k, w, (a, b, c), ScramblerSpec kwargs)
CUSTOM = [
    ("xoroshiro128plus-2016", "xoroshiro", 2, 64, (55, 14, 36), dict(kind="plus", word_i=0, word_j=1)),
    ("xoroshiro1024pp17", "xoroshiro", 16, 64, (25, 27, 36), dict(kind="plusplus", word_i=0, word_j=15, R=17)),
    ("xoshiro256ss-w0", "xoshiro", 4, 64, (17, 45, None), dict(kind="starstar", word_i=0, S=5, R=7, T=9)),
    ("xoshiro256-a11b50-plus12", "xoshiro", 4, 64, (11, 50, None), dict(kind="plus", word_i=1, word_j=2)),
    ("xoshiro512star", "xoshiro", 8, 64, (11, 21, None), dict(kind="star", word_i=1, S=0x9E3779B97F4A7C13)),
    ("xorshift128plus-23-18-5", "xorshift", 2, 64, (23, 18, 5), dict(kind="plus", word_i=0, word_j=1)),
    ("xoroshiro64ss-27-10-14", "xoroshiro", 2, 32, (27, 10, 14), dict(kind="starstar", word_i=0, S=0x9E3779BB, R=5, T=5)),
    ("xoshiro128pp-r9-12", "xoshiro", 4, 32, (9, 11, None), dict(kind="plusplus", word_i=1, word_j=2, R=9)),
    ("xoshiro256x32ss", "xoshiro", 8, 32, (9, 11, None), dict(kind="starstar", word_i=1, S=5, R=7, T=9)),
    ("xorshift64-5-7-3", "xorshift", 2, 32, (5, 7, 3), dict(kind="none", word_i=0)),
    # a shape without device kernels (host algebra only; device calls raise)
    ("xoroshiro256-4w", "xoroshiro", 4, 64, (24, 16, 37), dict(kind="plus", word_i=0, word_j=3)),
]


def hx(v):
    return f"0x{int(v):x}"


def main():
    out = {}
    for name, fam, k, w, (a, b, c), sck in CUSTOM:
        spec = custom_spec(fam, k, w, a, b, c, scrambler=ScramblerSpec(**sck), name=name)
        n = spec.kind.n
        d = {"family": fam, "k": k, "w": w, "a": a, "b": b, "c": c, "scrambler": sck,
             "char_poly": hx(engine_char_poly(spec).bits),
             "jump_poly": hx(compute_jump_poly(spec, 1 << (n // 2)).poly.bits)}
        g = Generator.from_seed(spec, 42)
        d["first_outputs_seed42"] = [hx(g.next()) for _ in range(100)]
        ls = LanedStream(spec, seed=42, lanes=40, lane_len=1 << (n // 2))
        st = VecStepper(spec.kind, spec.params)
        S = ls.S.copy()
        d["substreams"] = [[hx(x) for x in st.flat(S)[:, i]] for i in range(40)]
        for _ in range(64):
            st.step(S)
        fl = st.flat(S)
        d["substreams_after_64"] = [[hx(x) for x in fl[:, i]] for i in range(40)]
        d["laned_3000"] = [hx(x) for x in np.concatenate(list(output_stream(spec, 42, 3000, lanes=5, lane_len=512)))]
        out[name] = d
        print(name, "ok", flush=True)
    with open(os.path.join(HERE, "custom.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()

"""Golden HWD reports produced by the REFERENCE (slprng.hwd.run_generator),
for the GPU HWD consumer's parity tests.  Build-container only (imports
/root/reference); the JSON it writes is committed.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_hwd.py [--slow]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
from slprng import hwd  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # name, seed, checkpoint_start, config kwargs
    ("xoshiro256starstar", 3, 60_000, dict(w=64, k=4, byte_limit=8 * 200_000)),
    ("xoshiro256plus", 1, 1_000_000, dict(w=64, k=8, byte_limit=8 * 10_000_000)),
    ("xoroshiro128plus", 5, 500_000, dict(w=64, k=6, byte_limit=8 * 4_000_000, mode="transitional")),
    ("xoshiro128plus", 2, 1_000_000, dict(w=32, k=8, byte_limit=4 * 8_000_000)),
    ("xoroshiro64star", 9, 250_000, dict(w=32, k=5, byte_limit=4 * 3_000_000, mode="transitional")),
    ("xoshiro256starstar", 4, 300_000, dict(w=32, k=6, byte_limit=8 * 2_000_000, split=True)),
    ("xorshift128plus", 1, 1_000_000, dict(w=64, k=8, byte_limit=8 * 30_000_000, mode="transitional")),
]
SLOW = [
    # the paper rows of test_hwd.py:286-304
    ("xorshift128plus", 1, None, dict(w=64, k=8, byte_limit=int(2.4e10), batch_size=2_300_000, mode="transitional")),
    ("xoshiro256starstar", 1, None, dict(w=64, k=8, byte_limit=int(1e10), batch_size=2_300_000)),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true")
    args = ap.parse_args()
    path = os.path.join(HERE, "hwd.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name, seed, cps, kw in CASES + (SLOW if args.slow else []):
        key = f"{name}/{seed}/{cps}/" + ",".join(f"{k}={v}" for k, v in sorted(kw.items()))
        if key in out:
            continue
        t0 = time.time()
        cfg = hwd.HwdConfig(**kw)
        rep = hwd.run_generator(name, cfg, seed=seed, checkpoint_start=cps, lanes=16384, lane_len=1024)
        d = rep.to_dict()
        d.update({"name": name, "seed": seed, "checkpoint_start": cps, "config": kw,
                  "ref_seconds": round(time.time() - t0, 1)})
        out[key] = d
        print(key, d["status"], d["values"], d["p_value"], d["signature"], d["ref_seconds"], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

"""output_stream host path: per-chunk wall time and whether the chunk was a
pooled DMA target; 2^30 values, 2^16 lanes x 1024 (the bench geometry)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402

spec = P.get_spec("xoshiro256starstar")
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
for rep in range(2):
    t0 = time.perf_counter()
    times, pooled = [], 0
    last = t0
    got = 0
    for c in P.output_stream(spec, 42, 1 << 30, lanes=lanes, lane_len=1024):
        now = time.perf_counter()
        times.append(round((now - last) * 1e3, 1))
        last = now
        pooled += isinstance(c.base, torch.Tensor)
        got += c.size
    dt = time.perf_counter() - t0
    print(json.dumps({"rep": rep, "lanes": lanes, "values_per_s": got / dt, "pooled": pooled, "chunks": len(times),
                      "ms_per_chunk": times}), flush=True)

"""Store-path experiments (round 1): write-bandwidth ceilings and how the
stream-major TMA fill depends on row length / layout.  Prints JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


GB = 1 << 30
buf = torch.empty(8 * GB, dtype=torch.uint8, device="cuda")
for label, fn in [("torch_fill_u8", lambda: buf.fill_(1)), ("torch_zero", lambda: buf.zero_()),
                  ("torch_fill_i64", lambda: buf.view(torch.int64).fill_(7))]:
    ms = timeit(fn)
    print(json.dumps({"exp": label, "ms": ms, "GBps": 8 * GB / ms / 1e6}), flush=True)
src = torch.empty(4 * GB, dtype=torch.uint8, device="cuda")
ms = timeit(lambda: buf[: 4 * GB].copy_(src))
print(json.dumps({"exp": "torch_copy_4GiB", "ms": ms, "GBps(read+write)": 8 * GB / ms / 1e6}), flush=True)
del buf, src

spec = P.get_spec(os.environ.get("GEN", "xoshiro256starstar"))
for n, T in [(1 << 20, 1024), (1 << 17, 8192), (1 << 24, 64), (1 << 22, 256), (1 << 14, 65536)]:
    sub = D.Substreams.from_seed(spec, 42, n)
    for layout in ("stream", "position"):
        out = torch.empty((n, T) if layout == "stream" else (T, n), dtype=torch.uint64, device="cuda")
        ms = timeit(lambda: sub.fill(T, out=out, layout=layout))
        print(json.dumps({"exp": f"fill_{layout}", "n": n, "T": T, "ms": ms,
                          "GBps": n * T * 8 / ms / 1e6, "store_path": os.environ.get("SLP_STORE_PATH", "0")}),
              flush=True)
        del out

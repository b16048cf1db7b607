"""Few long substreams (segment split, device._fill_split): total fill time of
n substreams x T outputs, and its parts -- the split jump
(slp_split_substreams) alone and the segment fill alone -- warm, CUDA events.
One JSON line per (generator, n, T)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import _native  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

CASES = [(1, 1 << 28), (16, 1 << 24), (1000, 1 << 18), (1 << 12, 1 << 16), (1 << 20, 1 << 10),
         (1 << 17, 1 << 13), (1 << 18, 1 << 13), (1 << 19, 1 << 12), (1 << 20, 1 << 11),  # long rows, no split
         (1 << 17, 1 << 14), (1 << 16, 1 << 15), (3 << 15, 1 << 14), (1 << 17, 3 << 13)]  # row strides 2^17+
NAMES = [a for a in sys.argv[1:] if not a.startswith("--")] or ["xoshiro256starstar", "xoroshiro128plus",
                                                                  "xoroshiro1024starstar"]
# The --sweep of split parameters in profiles/round1_split.jsonl (target
# threads, min segment, segment per state bit) ran on the Python-side
# prototype of the split; the chosen values (2^18, 2048, 8) now live in the
# C ABI (slp_split_factor), so this script times the library as built.
SWEEP = [None]


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for name, sw_par in [(a, b) for a in NAMES for b in SWEEP]:
    spec = P.get_spec(name)
    gid = D.native_id(spec)
    L = _native.lib()
    for n, T in CASES:
        sub = D.Substreams.from_seed(spec, 42, n)
        out = torch.empty((n, T), dtype=torch.uint64, device="cuda")
        res = {"name": name, "n": n, "T": T, "split_params": sw_par}
        ms = timeit(lambda: D.fill(spec, sub.states, T, out=out))
        res["fill_ms"] = ms
        res["TB_s"] = n * T * 8 / ms / 1e9
        J = D._split_factor(spec, n, T, "stream", T)
        res["J"] = J
        if J > 1:
            seg = torch.empty((spec.kind.k, n * J), dtype=sub.states.dtype, device="cuda")
            sw, sn = _native.int_to_words(T // J)
            stream = D._stream_ptr(seg.device)

            def split():
                _native.check(L.slp_split_substreams(gid, ctypes.c_void_p(sub.states.data_ptr()), n, n, sw, sn, J,
                                                     ctypes.c_void_p(seg.data_ptr()), n * J, stream), "split")
            res["split_ms"] = timeit(split)
            res["seg_fill_ms"] = timeit(lambda: D.fill(spec, seg, T // J, out=out.view(n * J, T // J),
                                                      advance=False))
        print(json.dumps(res), flush=True)

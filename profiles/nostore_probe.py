"""Is k_fill store-bound or generation-bound?  Times the fill of BASELINE
config shapes with and without the TMA stores, with the median SM clock
during the timed launches (NVML).  The store-less kernel is a variant build
(round 2 measured it through an environment switch, since removed so that
no run-time setting can drop stores):

  make variant VARIANT=nostore EXTRA=-DSLP_MEASURE_NO_STORE
  python profiles/nostore_probe.py [cases] [launches]
  SLP_LIB=variants/libslp_nostore.so python profiles/nostore_probe.py ...
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_1805_01407_b200 as P  # noqa: E402
from paper_1805_01407_b200 import device as D  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from pace_sweep import CASES  # noqa: E402


def main():
    cases = (sys.argv[1] if len(sys.argv) > 1 else "c2,c4,c3").split(",")
    launches = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for case in cases:
        gen, n, T, kind, layout = CASES[case][:5]
        spec = P.get_spec(gen)
        sub = D.Substreams.from_seed(spec, 42, n)
        out = sub.fill(T, kind=kind, layout=layout)
        nbytes = out.numel() * out.element_size()
        for _ in range(5):
            sub.fill(T, kind=kind, layout=layout, out=out)
        torch.cuda.synchronize()
        clocks, stop = [], threading.Event()

        def sample():
            while not stop.is_set():
                clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                time.sleep(0.005)

        th = threading.Thread(target=sample)
        th.start()
        ev0.record()
        for _ in range(launches):
            sub.fill(T, kind=kind, layout=layout, out=out)
        ev1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = ev0.elapsed_time(ev1) / launches
        clocks.sort()
        print(json.dumps({"case": case, "lib": os.environ.get("SLP_LIB", "in-tree"),
                          "pace_gbps": P._native.lib().slp_set_fill_pace(-1), "ms": round(ms, 4),
                          "GBps_equiv": round(nbytes / ms / 1e6, 1),
                          "sm_mhz_median": clocks[len(clocks) // 2] if clocks else None}), flush=True)
        del out, sub
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""Round 2 A/B: the stock reference (baseline/_ref/slprng)
against the numpy port that round 1 timed (oracle/cpu_baseline.py), on the
same host cores and config-2 work (xoshiro256**, seed 42, 2^20 substreams x
1024 outputs per step).  Three figures, outputs/s:
  stock_resident     lane set-up once, then each step = 1024 x (apply_vec,
                     VecStepper.step) per substream (bench.py --impl reference)
  stock_setup_each   the same step plus the stock set-up redone every step
                     (Generator.jump + LanedStream, generators.py:315-334, 435-463)
  port_setup_each    round 1's port: set-up + step in one task per slice
One JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.cpu_baseline import CpuBaseline  # noqa: E402
from oracle.ref_baseline import ReferenceArm  # noqa: E402

N, T = 1 << 20, 1024
res = {"cores": os.cpu_count()}
arm = ReferenceArm("xoshiro256starstar", 42, N, T)
try:
    _, _, s, x = arm.step(checksum=True)
    secs = [arm.step()[1] for _ in range(3)]
finally:
    arm.close()
res["stock_setup_s"] = round(arm.init_wall_s, 3)
res["stock_resident"] = N * T / (sum(secs) / 3)
res["stock_setup_each"] = N * T / (sum(secs) / 3 + arm.init_wall_s)
res["stock_checksum"] = [hex(s), hex(x)]
cb = CpuBaseline("xoshiro256starstar", 42, T)
try:
    per = N // cb.procs
    t0 = time.perf_counter()
    n, dt = cb.step(per)
    res["port_setup_each"] = n / dt
    res["port_sample"] = f"{cb.procs} procs x {per} substreams (one config-2 step)"
finally:
    cb.close()
res["stock_over_port_setup_each"] = res["stock_setup_each"] / res["port_setup_each"]
print(json.dumps(res))

import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(reps): fn()
        e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best
for name in ["xoroshiro1024plusplus", "xoshiro512starstar", "xoshiro256starstar", "xoroshiro128plus", "xoshiro128plusplus"]:
    spec = P.get_spec(name)
    r = {"lib": os.path.basename(os.environ.get("SLP_LIB") or "main"), "name": name}
    for n in (1 << 17, 1 << 20, 1 << 21):
        r["init_%d" % n] = round(timeit(lambda: D.Substreams.from_seed(spec, 42, n)), 4)
    print(json.dumps(r), flush=True)

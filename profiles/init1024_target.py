import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import device as D
spec = P.get_spec("xoroshiro1024starstar")
for _ in range(3):
    D.Substreams.from_seed(spec, 42, 1 << 15)
torch.cuda.synchronize()

"""Short HWD run for ncu (k_hwd): xoshiro256** k=8, 8e9 bytes, one checkpoint."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_01407_b200 import hwd  # noqa: E402

cfg = hwd.HwdConfig(w=64, k=8, byte_limit=8 * 10 ** 9)
rep = hwd.run_generator("xoshiro256starstar", cfg, seed=1, checkpoint_start=10 ** 9)
print(rep.status, rep.values, rep.p_value)

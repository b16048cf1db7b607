"""Stream-major rows that are not 16-byte aligned (row-group TMA, FILL_TMA_G)
against aligned rows, several generators and T; one JSON line each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "slow_shapes.py")).read().split("N = 1 << 20")[0])
N = 1 << 20
for name in ("xoshiro256starstar", "xoroshiro128plus", "xoshiro512starstar"):
    for T in (1024, 1023, 2047, 1001):
        case("sm", name, N, T)
case("sm u32", "xoshiro128starstar", 2 * N, 1024)
case("sm u32", "xoshiro128starstar", 2 * N, 1023)
case("sm u32", "xoshiro128starstar", 2 * N, 1022)

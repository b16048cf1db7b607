import json, os, sys
sys.path.insert(0, "/root/repo")
sys.argv = [sys.argv[0]]
exec(open("/root/repo/profiles/slow_shapes.py").read().split("N = 1 << 20")[0])
N = 1 << 20
case("pm aligned", "xoshiro256starstar", N, 1024, "position")
case("pm odd", "xoshiro256starstar", N + 1, 1024, "position")
case("pm aligned u32", "xoshiro128starstar", 2 * N, 1024, "position")
case("pm odd u32", "xoshiro128starstar", 2 * N + 1, 1024, "position")

for v in spt4 spt2 spt1; do echo "== $v"; SLP_LIB=variants/libslp_$v.so python profiles/init_bench.py xoroshiro128plus xoshiro256starstar xoshiro512starstar xoroshiro1024starstar xoshiro128starstar | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['name'][:22].ljust(22), 'tables %.3f ms  8x2^18 %.3f ms' % (d['init_ms_tables'], d['init_ms_8x2^18_tables']))
"; done

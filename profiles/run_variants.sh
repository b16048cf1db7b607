# A/B: run the microbenchmark against each variants/libslp_*.so
for v in variants/libslp_*.so; do
  echo "== $v"
  SLP_LIB=$v python profiles/microbench.py ${GENS:-xoshiro256starstar xoshiro256plusplus xoroshiro128plus xoshiro512starstar xoroshiro1024starstar xoshiro128starstar} --reps ${REPS:-10} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['name'][:22].ljust(22), 'store %.3g'%d.get('store_out_per_s',0), 'int %.3g'%d['fused_int_out_per_s'], 'exact %.3g'%d['fused_exact_out_per_s'], 'f64 %.3g'%d['fused_f64_out_per_s'], 'init %.3f'%d['init_ms'])
"
done

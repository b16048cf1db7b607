# f64 conversion as (x & ~0x7FF) * 2^-64 (variants/libslp_f64a.so) vs (x >> 11) * 2^-53 (in-tree build)
SLP_LIB=variants/libslp_f64a.so timeout 900 python -m pytest tests/test_gpu_fill_kinds.py tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x 2>&1 | tail -2
C="--cfg main:6500 --cfg variants/libslp_f64a.so:6500 --cfg main:0 --cfg variants/libslp_f64a.so:0"
for case in ${CASES:-c2f64 c3}; do
  timeout 300 python profiles/ab_pace.py --case $case --rounds ${ROUNDS:-8} --launches 30 $C
done

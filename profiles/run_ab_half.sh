# half-tile TMA stores (variants/libslp_half.so, -DSLP_FILL_HALF=1) vs the in-tree build: parity, then interleaved A/B
SLP_LIB=variants/libslp_half.so timeout 900 python -m pytest tests/test_gpu_fill_kinds.py tests/test_gpu_pacing.py tests/test_gpu_parity.py tests/test_gpu_split.py -q -x 2>&1 | tail -2
C="--cfg main:6500 --cfg variants/libslp_half.so:6500 --cfg variants/libslp_half.so:6700 --cfg main:6700 --cfg main:0 --cfg variants/libslp_half.so:0"
for case in ${CASES:-c2 c4 c3 c2f64}; do
  timeout 300 python profiles/ab_pace.py --case $case --rounds ${ROUNDS:-8} --launches 50 $C
done

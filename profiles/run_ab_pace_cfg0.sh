# pacing target sweep for the unroll-32 fill configuration (variants/libslp_cfg0.so)
L=variants/libslp_cfg0.so
C="--cfg main:0 --cfg $L:0 --cfg $L:6200 --cfg $L:6400 --cfg $L:6500 --cfg $L:6600 --cfg $L:6700 --cfg $L:6800 --cfg $L:7000"
for case in ${CASES:-c2 c4 c3 c2f64 x1024}; do
  timeout 300 python profiles/ab_pace.py --case $case --rounds ${ROUNDS:-10} $C
done

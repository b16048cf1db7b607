# interleaved A/B of library builds x store-pacing targets (profiles/ab_pace.py)
C="--cfg main:0 --cfg main:6000 --cfg main:6200 --cfg main:6400 --cfg main:6600 --cfg variants/libslp_w14.so:0 --cfg variants/libslp_w14.so:6000 --cfg variants/libslp_w14.so:6200 --cfg variants/libslp_w14.so:6400 --cfg variants/libslp_w14.so:6600 --cfg variants/libslp_w9.so:6200 --cfg variants/libslp_w9.so:6400"
for case in ${CASES:-c2 c4 c3}; do
  timeout 300 python profiles/ab_pace.py --case $case --rounds ${ROUNDS:-12} $C
done

# pacing wait: spin on %globaltimer (spinold) vs __nanosleep (spin = new code), interleaved
C="--cfg variants/libslp_spinold.so:6500 --cfg variants/libslp_spin.so:6500 --cfg variants/libslp_spinold.so:0 --cfg variants/libslp_spin.so:6800"
for case in ${CASES:-c2 c4 x1024}; do
  timeout 300 python profiles/ab_pace.py --case $case --rounds ${ROUNDS:-8} --launches 50 $C
done

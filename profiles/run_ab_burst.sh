# store pacing: catch-up window (SLP_FILL_PACE_BURST) x target, in-tree build (unroll-32 tiles)
C="--cfg main:0 --cfg main:6400:1 --cfg main:6400:2 --cfg main:6400:4 --cfg main:6600:1 --cfg main:6600:2 --cfg main:6600:4 --cfg main:6600:8 --cfg main:6800:2 --cfg main:6800:4"
for case in ${CASES:-c2 c4 c3}; do
  timeout 300 python profiles/ab_pace.py --case $case --rounds ${ROUNDS:-10} $C
done

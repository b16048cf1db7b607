# generation-side A/B on config 2 (profiles/ab_pace.py): store batching (nbN),
# (SLP_FILL_NO_STORE was a run-time switch when this ran; now: a build with -DSLP_MEASURE_NO_STORE)
# no shared stores (nosts), unroll-32 tiles (cfg0); with and without the TMA stores
C="--cfg main:0 --cfg variants/libslp_nb2.so:0 --cfg variants/libslp_nb4.so:0 --cfg variants/libslp_nb8.so:0 --cfg variants/libslp_nosts.so:0 --cfg variants/libslp_cfg0.so:0 --cfg main:6400 --cfg variants/libslp_nb4.so:6400 --cfg variants/libslp_cfg0.so:6400"
echo '{"note": "with stores"}'
timeout 300 python profiles/ab_pace.py --case c2 --rounds 10 $C
echo '{"note": "SLP_FILL_NO_STORE=1"}'
SLP_FILL_NO_STORE=1 timeout 300 python profiles/ab_pace.py --case c2 --rounds 10 $C

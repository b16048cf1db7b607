# fill-configuration tuning under store pacing (round 2): every cfg variant x
# (SLP_FILL_NO_STORE was a run-time switch when this ran; now: a build with -DSLP_MEASURE_NO_STORE)
# (generator, kind), paced at the candidate default, generation-only, unpaced
SLP_FILL_PACE_GBPS=${PACE:-6500} python profiles/tune_fill.py run > gpurun_out/tune_paced.jsonl 2> gpurun_out/tune_paced.err
SLP_FILL_NO_STORE=1 python profiles/tune_fill.py run > gpurun_out/tune_gen.jsonl 2> gpurun_out/tune_gen.err
SLP_FILL_PACE_GBPS=0 python profiles/tune_fill.py run > gpurun_out/tune_unpaced.jsonl 2> gpurun_out/tune_unpaced.err

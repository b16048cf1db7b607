set -x
python bench.py --extra > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_full.err
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_small.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
python profiles/ncu_target.py > gpurun_out/target.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fill -s 1 -c 1 -o gpurun_out/prof_fill python profiles/ncu_target.py > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/prof_fused python profiles/ncu_target.py > gpurun_out/ncu_full2.log 2>&1; echo "ncu3 rc=$?"

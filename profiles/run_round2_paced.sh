# Round-2 re-measurement after store pacing + the re-tuned fill table:
# GPU tests, smoke, bench, ncu launch list of the bench and a full capture of k_fill / k_fused
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu_p.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_p.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_p.txt
timeout 900 python bench.py > gpurun_out/bench_p.json 2> gpurun_out/bench_p.err; echo "bench rc=$?"
python bench.py --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-extra > gpurun_out/b_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
python profiles/ncu_target.py > gpurun_out/target.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'k_fill|k_fused$' -s 2 -c 2 \
  -o gpurun_out/prof_p python profiles/ncu_target.py > gpurun_out/ncu_full_p.log 2>&1; echo "ncu-full rc=$?"

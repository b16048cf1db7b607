# Round-2 measurement: parity tests, smoke, bench (ours + reference arm),
# ncu launch list of the bench command and full captures of the top kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
python bench.py --steps 100 --warmup 10 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_r2.json 2> gpurun_out/bench_ref_r2.err; echo "ref rc=$?"
python bench.py --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
  python bench.py --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
python profiles/ncu_target.py > gpurun_out/target.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'k_fill|k_fused$' -s 2 -c 2 \
  -o gpurun_out/prof_r2 python profiles/ncu_target.py > gpurun_out/ncu_full_r2.log 2>&1; echo "ncu-full rc=$?"
python profiles/ref_vs_port.py > gpurun_out/ref_vs_port_r2.json 2> gpurun_out/ref_vs_port_r2.err; echo "ref_vs_port rc=$?"

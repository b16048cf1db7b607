# Round-2 final measurement of the current build: GPU tests (with skip reasons),
# smoke, bench (both arms), ncu launch list of the bench and a full capture of k_fill / k_fused
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/final_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1 | tail -25 > gpurun_out/final_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.txt
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err; echo "ref rc=$?"
python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extra > gpurun_out/final_b_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extra > gpurun_out/final_ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
python profiles/ncu_target.py > gpurun_out/final_target.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'k_fill|k_fused$' -s 2 -c 2 \
  -o gpurun_out/final_prof python profiles/ncu_target.py > gpurun_out/final_ncu_full.log 2>&1; echo "ncu-full rc=$?"

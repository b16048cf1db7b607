# parity + per-kernel timings + ncu of the fill kernel (round 1, iteration b)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -5
python profiles/microbench.py xoshiro256starstar xoshiro256plus xoshiro256plusplus xoroshiro128plus xoshiro128starstar xoroshiro1024starstar xoshiro512starstar > gpurun_out/micro_b.jsonl 2>&1; echo "micro rc=$?"
cat gpurun_out/micro_b.jsonl
python profiles/ncu_target.py > gpurun_out/target.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fill -s 1 -c 1 -o gpurun_out/prof_fill_b python profiles/ncu_target.py > gpurun_out/ncu_full_b.log 2>&1; echo "ncu rc=$?"

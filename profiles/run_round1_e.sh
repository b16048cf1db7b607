mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --steps 50 --warmup 5 --extra --no-cpu-baseline > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_e.err
python -c "import json; d=json.load(open('gpurun_out/bench_e.json')); print(json.dumps(d['extra'])); print(d['e2e_device_resident'])"
torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_trun.json 2> gpurun_out/bench_trun.err; echo "torchrun rc=$?"
tail -2 gpurun_out/bench_trun.err; cut -c1-300 gpurun_out/bench_trun.json

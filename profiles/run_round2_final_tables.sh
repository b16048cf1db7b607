# after the final fill table: GPU tests, configs 3/4, all generators, bench line
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu_f.txt
python profiles/configs_bench.py > gpurun_out/configs34_r2.jsonl 2> gpurun_out/configs34_r2.err
python profiles/microbench.py $(python -c "import paper_1805_01407_b200 as P; print(' '.join(P.registry_names(True)))") --reps 10 > gpurun_out/micro_all_r2.jsonl 2> gpurun_out/micro_all_r2.err
timeout 900 python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo "bench rc=$?"

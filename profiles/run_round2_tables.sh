# round-2 throughput tables with store pacing: configs 3/4 at full size, all generators, slow shapes, ragged rows
python profiles/configs_bench.py > gpurun_out/configs34_r2.jsonl 2> gpurun_out/configs34_r2.err
python profiles/microbench.py --reps 10 > gpurun_out/micro_r2.jsonl 2> gpurun_out/micro_r2.err
python profiles/slow_shapes.py > gpurun_out/slow_shapes_r2.jsonl 2> gpurun_out/slow_shapes_r2.err
python profiles/ragged_bench.py > gpurun_out/ragged_r2.jsonl 2> gpurun_out/ragged_r2.err

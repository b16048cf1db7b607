mkdir -p gpurun_out
python profiles/store_experiments.py > gpurun_out/store_exp.jsonl 2>&1; echo rc=$?
SLP_STORE_PATH=2 python profiles/store_experiments.py 2>&1 | grep fill_stream >> gpurun_out/store_exp.jsonl
cat gpurun_out/store_exp.jsonl

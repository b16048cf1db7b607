# per-row bulk-copy path for unaligned stream-major rows (k_fill_rows): parity, then A/B vs row-group TMA
timeout 1200 python -m pytest tests/test_gpu_fill_kinds.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_pacing.py tests/test_gpu_split.py tests/test_gpu_custom.py -q -x 2>&1 | tail -3
for rb in 1 0; do SLP_ROW_BULK=$rb RAGGED_TS=1023,1055,2047,1027,1537 python profiles/ragged_bench.py | sed "s/^{/{\"row_bulk\": $rb, /"; done > gpurun_out/rows_ragged.jsonl 2>&1

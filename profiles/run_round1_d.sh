mkdir -p gpurun_out
python profiles/ncu_target.py > gpurun_out/target.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_fused -s 1 -c 1 -o gpurun_out/prof_fused_d python profiles/ncu_target.py > gpurun_out/ncu_fused_d.log 2>&1; echo "ncu rc=$?"

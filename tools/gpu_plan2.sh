cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/plan_time.py > gpurun_out/${TAG}_plan.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "plan" >> gpurun_out/${TAG}_plan.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plan_fused -s 37 -c 1 -o gpurun_out/${TAG}_plan python tools/plan_time.py > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_plan.ncu-rep > gpurun_out/${TAG}_ncu_plan.txt 2>&1; rm -f gpurun_out/${TAG}_plan.ncu-rep

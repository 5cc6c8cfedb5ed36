cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/plan_time.py > gpurun_out/${TAG}_plan_time.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plan_hist -s 14 -c 1 -o gpurun_out/${TAG}_plan_C3 python tools/plan_time.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_plan_C3.ncu-rep > gpurun_out/${TAG}_ncu_plan_C3.txt 2>&1 && rm -f gpurun_out/${TAG}_plan_C3.ncu-rep

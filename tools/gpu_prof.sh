cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/loop_probe.py C3 C4 > gpurun_out/${TAG}_loop_probe.txt 2>&1
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_csr -s 2 -c 1 \
    -o gpurun_out/${TAG}_csr python tools/csr_time.py 3 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_csr.ncu-rep > gpurun_out/${TAG}_ncu_csr.txt 2>&1
python tools/run_solve_once.py C3 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${TAG}_loop_C3 python tools/run_solve_once.py C3 > gpurun_out/${TAG}_ncu_loop.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_loop_C3.ncu-rep > gpurun_out/${TAG}_ncu_loop_C3.txt 2>&1; rm -f gpurun_out/${TAG}_loop_C3.ncu-rep

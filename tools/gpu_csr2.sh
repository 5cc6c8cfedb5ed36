cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "csr or C5 or routing" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python tools/csr_time.py > gpurun_out/${TAG}_csr.txt 2>&1
CSK_CSR_GATHER=1 timeout 300 python tools/csr_time.py >> gpurun_out/${TAG}_csr.txt 2>&1
timeout 600 nsys 2>/dev/null; CSK_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 8 -c 12 --csv python tools/csr_time.py 3 > gpurun_out/${TAG}_csr_launches.csv 2>&1
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_csr_fold -s 1 -c 1 -o gpurun_out/${TAG}_fold python tools/csr_time.py 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_fold.ncu-rep > gpurun_out/${TAG}_ncu_fold.txt 2>&1; rm -f gpurun_out/${TAG}_fold.ncu-rep

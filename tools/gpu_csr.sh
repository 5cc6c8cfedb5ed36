cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "csr or C5" > gpurun_out/p6_pytest.log 2>&1; echo "exit $?" >> gpurun_out/p6_pytest.log
timeout 300 python tools/csr_time.py > gpurun_out/p6_csr.txt 2>&1
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_csr -s 2 -c 1 \
    -o gpurun_out/p6_csr python tools/csr_time.py 3 > gpurun_out/p6_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p6_csr.ncu-rep > gpurun_out/p6_ncu_csr.txt 2>&1
tail -3 gpurun_out/p6_pytest.log

cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "csr or residual or small_configs or C3_full or launch_shapes or C5" > gpurun_out/p2_pytest.log 2>&1; echo "exit $?" >> gpurun_out/p2_pytest.log
timeout 300 python tools/csr_time.py > gpurun_out/p2_csr.txt 2>&1
CSK_L2_FETCH_GRAN=32 timeout 300 python tools/csr_time.py > gpurun_out/p2_csr_g32.txt 2>&1
timeout 600 python tools/loop_ab.py paper_2004_02480_b200/libcsk_r2a.so paper_2004_02480_b200/libcsk.so > gpurun_out/p2_ab.txt 2>&1
tail -3 gpurun_out/p2_pytest.log

cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=paper_2004_02480_b200/libcsk.so
timeout 900 python tools/loop_ab.py $L $L:CSK_LOOP_EXP=2 $L:CSK_LOOP_EXP=32 --configs=C2,C3,C4 > gpurun_out/${TAG}_ab.txt 2>&1
timeout 300 python tools/csr_time.py > gpurun_out/${TAG}_csr.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "csr" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log

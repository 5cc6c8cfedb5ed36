cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-sk}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sketch or C3 or C4 or plan" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
for i in 1 2; do
for v in ${LIBS:-libcsk_base.so libcsk.so}; do
echo "== $v" >> gpurun_out/${T}_time.txt
CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/sketch_kernel_time.py C3 C4 300000x100 700000x150 >> gpurun_out/${T}_time.txt 2>&1
CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/sketch_time.py C3 >> gpurun_out/${T}_time.txt 2>&1
done
done

cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-nrm}
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "norms or sketch" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
CSK_LIB=checked timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "norms" > gpurun_out/${T}_checked.log 2>&1; echo "exit $?" >> gpurun_out/${T}_checked.log
for i in 1 2; do
for v in ${LIBS}; do
echo "== $v" >> gpurun_out/${T}_time.txt
CSK_LIB=paper_2004_02480_b200/$v timeout 120 python tools/norms_time.py >> gpurun_out/${T}_time.txt 2>&1
done
done

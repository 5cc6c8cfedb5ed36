cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-ws}
CSK_LIB=checked timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "csr" > gpurun_out/${T}_checked.log 2>&1; echo "exit $?" >> gpurun_out/${T}_checked.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "csr or C5 or routing" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
for v in ${LIBS:-libcsk_base.so libcsk.so}; do
  echo "== $v" >> gpurun_out/${T}_csr_ab.txt
  CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/csr_time.py 4 >> gpurun_out/${T}_csr_ab.txt 2>&1
done

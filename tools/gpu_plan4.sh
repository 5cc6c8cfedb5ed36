cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-pl}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "plan or sketch or csr or C3 or C5 or routing or hash or map" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
CSK_LIB=checked timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "plan or map or hash" > gpurun_out/${T}_checked.log 2>&1; echo "exit $?" >> gpurun_out/${T}_checked.log
timeout 600 python tests/fuzz_parity.py 200 777 > gpurun_out/${T}_fuzz.log 2>&1; echo "exit $?" >> gpurun_out/${T}_fuzz.log
for i in 1 2; do
for v in libcsk_base.so libcsk.so; do
echo "== $v" >> gpurun_out/${T}_time.txt
CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/plan_time.py >> gpurun_out/${T}_time.txt 2>&1
CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/sketch_time.py C3 >> gpurun_out/${T}_time.txt 2>&1
CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/csr_time.py 3 >> gpurun_out/${T}_time.txt 2>&1
done
done

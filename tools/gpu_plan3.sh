cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "plan or sketch or hash or csr or small_configs or identity or routing or virtual" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python tools/plan_time.py > gpurun_out/${TAG}_plan.txt 2>&1
CSK_PLAN_ATOMIC=1 timeout 300 python tools/plan_time.py >> gpurun_out/${TAG}_plan.txt 2>&1
timeout 300 python tools/sketch_time.py C3 C4 >> gpurun_out/${TAG}_plan.txt 2>&1
timeout 300 python tools/csr_time.py >> gpurun_out/${TAG}_plan.txt 2>&1

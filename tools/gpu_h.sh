cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 800 python tools/loop_ab.py ab/libcsk_base.so ab/libcsk_f2.so ab/libcsk_h.so --configs=C2,C3,C4,C5 > gpurun_out/${TAG}_ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log

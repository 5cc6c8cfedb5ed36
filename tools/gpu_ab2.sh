cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
B=paper_2004_02480_b200/libcsk_base.so
L=paper_2004_02480_b200/libcsk.so
timeout 900 python tools/loop_ab.py $B $L $B $L --configs=${CFGS:-C2,C3,C4} > gpurun_out/${TAG}_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "${PYK:-solve or C3 or lockstep or mwrk}" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log

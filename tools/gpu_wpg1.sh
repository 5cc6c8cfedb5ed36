cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=paper_2004_02480_b200/libcsk.so
timeout 600 python tools/loop_ab.py $L $L:CSK_LOOP_WPG=1 --configs=C3 > gpurun_out/${TAG}_ab.txt 2>&1
CSK_DEBUG=1 CSK_LOOP_WPG=1 timeout 120 python tools/run_solve_once.py C3 > gpurun_out/${TAG}_dbg.txt 2>&1

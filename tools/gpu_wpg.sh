cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=paper_2004_02480_b200/libcsk.so
timeout 900 python tools/loop_ab.py $L $L:CSK_FORCE_WPG=1 --configs=C3,C2 > gpurun_out/${TAG}_ab.txt 2>&1

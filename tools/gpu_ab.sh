cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 800 python tools/loop_ab.py $LIBS --configs=$CFGS > gpurun_out/${TAG}_ab.txt 2>&1

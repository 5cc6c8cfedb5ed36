cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CSK_LIB=$PWD/ab/libcsk_prof_gemv.so timeout 300 python tools/loop_probe.py C4 --ctas=148 > gpurun_out/${TAG}_probe.txt 2>&1

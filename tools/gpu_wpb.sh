cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-wpb}
for v in libcsk_base.so libcsk_wpbA.so libcsk_wpbB.so; do
echo "== $v" >> gpurun_out/${T}_time.txt
CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/sketch_kernel_time.py C3 300000x300 300000x400 200000x512 >> gpurun_out/${T}_time.txt 2>&1
CSK_WPB_MAX_N=512 CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/sketch_kernel_time.py C3 300000x300 300000x400 200000x512 >> gpurun_out/${T}_time.txt 2>&1
done
CSK_WPB_MAX_N=512 CSK_LIB=paper_2004_02480_b200/libcsk_wpbB.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sketch" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log

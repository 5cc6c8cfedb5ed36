cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-g4}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sketch or C3 or C4 or table" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
CSK_LIB=checked timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sketch" > gpurun_out/${T}_checked.log 2>&1; echo "exit $?" >> gpurun_out/${T}_checked.log
for i in 1 2; do
echo "== base" >> gpurun_out/${T}_time.txt
CSK_LIB=paper_2004_02480_b200/libcsk_base.so timeout 300 python tools/sketch_kernel_time.py C3 C4 300000x512 200000x1000 100000x2000 >> gpurun_out/${T}_time.txt 2>&1
echo "== g4 off" >> gpurun_out/${T}_time.txt
CSK_SKETCH_G4=0 timeout 300 python tools/sketch_kernel_time.py C3 C4 300000x512 200000x1000 100000x2000 >> gpurun_out/${T}_time.txt 2>&1
echo "== g4" >> gpurun_out/${T}_time.txt
timeout 300 python tools/sketch_kernel_time.py C3 C4 300000x512 200000x1000 100000x2000 >> gpurun_out/${T}_time.txt 2>&1
done

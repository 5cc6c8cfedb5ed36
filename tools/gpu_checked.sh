cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CSK_LIB=checked timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_checked_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_checked_pytest.log
CSK_LIB=checked timeout 600 python tools/sanitize_cases.py > gpurun_out/${TAG}_checked_cases.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_checked_cases.log
CSK_LIB=checked timeout 900 python tests/fuzz_parity.py 300 4242 > gpurun_out/${TAG}_checked_fuzz.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_checked_fuzz.log
timeout 300 python tools/sketch_time.py C3 C4 > gpurun_out/${TAG}_time.txt 2>&1
timeout 300 python tools/csr_time.py >> gpurun_out/${TAG}_time.txt 2>&1

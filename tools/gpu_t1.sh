cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python tools/table1.py --trials 50 --json gpurun_out/r02_table1.json > gpurun_out/r02_table1.md 2> gpurun_out/r02_table1.err
timeout 1800 python tests/fuzz_parity.py 800 20261020 > gpurun_out/r02_fuzz_parity.txt 2>&1; echo "exit $?" >> gpurun_out/r02_fuzz_parity.txt

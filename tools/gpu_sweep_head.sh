#!/bin/bash
# Randomised parity sweep (new seed) and the Table-1 protocol at HEAD:
# usage (under gpurun): bash tools/gpu_sweep_head.sh r02h
R=${1:-r02h}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python tests/fuzz_parity.py 600 20261021 > gpurun_out/${R}_fuzz_parity.txt 2>&1; echo "exit $?" >> gpurun_out/${R}_fuzz_parity.txt
timeout 2400 python tools/table1.py --trials 50 --json gpurun_out/${R}_table1.json > gpurun_out/${R}_table1.md 2>&1; echo "exit $?" >> gpurun_out/${R}_table1.md
tail -3 gpurun_out/${R}_fuzz_parity.txt; tail -5 gpurun_out/${R}_table1.md

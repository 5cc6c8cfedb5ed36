#!/bin/bash
# Full verification at HEAD: pytest -m gpu, smoke, bench (N=1), reference arm, ncu launch list.
# usage (under gpurun): bash tools/gpu_head.sh r02h
R=${1:-r02h}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${R}_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${R}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${R}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${R}_smoke.log
timeout 600 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${R}_launches.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
tail -3 gpurun_out/${R}_pytest_gpu.log; cat gpurun_out/${R}_smoke.log | tail -2; head -c 600 gpurun_out/${R}_bench.json

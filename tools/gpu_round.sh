#!/bin/bash
# One GPU session: the full-size parity artifacts (C4 50k, C5 to 1e-6; oracle minutes, on the
# host in the background), pytest -m gpu, then a bench line.  Output under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
PAR=${PAR:-1}
if [ "$PAR" = 1 ]; then
  timeout 2400 python tests/parity_full.py C5 --out gpurun_out/r02_parity_C5.txt > gpurun_out/parity_C5.log 2>&1 &
  P5=$!
  sleep 60
  timeout 2700 python tests/parity_full.py C4 --out gpurun_out/r02_parity_C4.txt > gpurun_out/parity_C4.log 2>&1 &
  P4=$!
  sleep 90
fi
timeout 2000 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
if [ "${BENCH:-1}" = 1 ]; then
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err
fi
if [ "$PAR" = 1 ]; then wait $P5; echo "C5 exit $?" >> gpurun_out/parity_C5.log; wait $P4; echo "C4 exit $?" >> gpurun_out/parity_C4.log; fi
tail -3 gpurun_out/pytest_gpu.log

#!/bin/bash
# L2-resident chunks at the front of each group's stream (SPREAD=0) or spread evenly with a
# per-group offset (SPREAD=1).  usage (under gpurun): bash tools/gpu_l2spread.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r02_l2spread_ab.txt
: > $O
for sp in 0 1; do for mb in ${L2PIN_LIST:-0 80 96 112 128}; do
  echo "== CSK_LOOP_L2PIN_SPREAD=$sp CSK_LOOP_L2PIN_MB=$mb" >> $O
  CSK_LOOP_L2PIN_SPREAD=$sp CSK_LOOP_L2PIN_MB=$mb CSK_LOOP_L2PIN_MINCHUNK=0 timeout 600 python tools/stream_time.py 200 >> $O 2>&1
done; done
cut -c1-75 $O

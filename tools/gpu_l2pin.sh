#!/bin/bash
# L2 residency sweep for the loop's streamed rows (CSK_LOOP_L2PIN_MB megabytes copied evict_last;
# CSK_LOOP_L2PIN_REST: the other rows evict_first (1) or unhinted (0)): C5 CSK loop and the MWRK
# (streamed A) cases of tools/stream_time.py.   usage (under gpurun): bash tools/gpu_l2pin.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/${L2PIN_OUT:-r02_l2pin_ab2.txt}
: > $O
for rest in ${L2PIN_REST_LIST:-0 1}; do
for mb in ${L2PIN_LIST:-0 64 96 112 128 160}; do
  echo "== CSK_LOOP_L2PIN_MB=$mb CSK_LOOP_L2PIN_REST=$rest" >> $O
  CSK_LOOP_L2PIN_REST=$rest CSK_LOOP_L2PIN_MB=$mb timeout 600 python tools/stream_time.py 200 >> $O 2>&1
done; done
cut -c1-75 $O

#!/bin/bash
# Whole-trajectory C4/C5 parity at HEAD (background, CPU oracle) beside the loop ncu captures and
# the phase probe: usage (under gpurun): bash tools/gpu_parity_head.sh r02h
R=${1:-r02h}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python tests/parity_full.py C4 --out gpurun_out/${R}_parity_C4.txt > gpurun_out/${R}_parity_C4.log 2>&1 &
P4=$!
sleep 45
timeout 2400 python tests/parity_full.py C5 --out gpurun_out/${R}_parity_C5.txt > gpurun_out/${R}_parity_C5.log 2>&1 &
P5=$!
sleep 60
python tools/run_solve_once.py C3 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${R}_loop_C3 python tools/run_solve_once.py C3 > /dev/null 2>&1
python tools/run_solve_once.py C4 2000 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${R}_loop_C4 python tools/run_solve_once.py C4 2000 > /dev/null 2>&1
for rep in gpurun_out/${R}_*.ncu-rep; do
    [ -f "$rep" ] || continue
    b=$(basename "$rep" .ncu-rep)
    python tools/ncu_summary.py "$rep" > "gpurun_out/${b/${R}_/${R}_ncu_}.txt" 2>&1 && rm -f "$rep"
done
wait $P4; echo "exit $?" >> gpurun_out/${R}_parity_C4.log
wait $P5; echo "exit $?" >> gpurun_out/${R}_parity_C5.log
timeout 600 python tools/loop_probe.py C3 C4 > gpurun_out/${R}_loop_probe.txt 2>&1
timeout 300 python tools/step_gaps.py C3 > gpurun_out/${R}_step_gaps.txt 2>&1
tail -2 gpurun_out/${R}_parity_C4.txt gpurun_out/${R}_parity_C5.txt
ls -la gpurun_out | grep ${R}

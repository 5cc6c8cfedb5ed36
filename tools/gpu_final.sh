#!/bin/bash
# Final evidence of the round (profile_round.sh minus Table 1, plus the whole-trajectory parity
# artifacts in the background): usage (under gpurun): bash tools/gpu_final.sh r02
R=${1:-r02}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python tests/parity_full.py C4 --out gpurun_out/${R}_parity_C4.txt > gpurun_out/${R}_parity_C4.log 2>&1 &
P4=$!
sleep 45
timeout 2400 python tests/parity_full.py C5 --out gpurun_out/${R}_parity_C5.txt > gpurun_out/${R}_parity_C5.log 2>&1 &
P5=$!
sleep 60
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${R}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${R}_pytest_gpu.log
wait $P4; echo "exit $?" >> gpurun_out/${R}_parity_C4.log
wait $P5; echo "exit $?" >> gpurun_out/${R}_parity_C5.log
timeout 1200 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
CSK_PROFILE_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches_C3.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-e2e \
    > gpurun_out/${R}_ncu_launches.log 2>&1
python tools/run_solve_once.py C3 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${R}_loop_C3 python tools/run_solve_once.py C3 > /dev/null 2>&1
python tools/run_solve_once.py C4 2000 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${R}_loop_C4 python tools/run_solve_once.py C4 2000 > /dev/null 2>&1
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_dense -s 2 -c 1 \
    -o gpurun_out/${R}_sketch_C3 python tools/sketch_time.py C3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plan_hist -s 14 -c 1 \
    -o gpurun_out/${R}_plan_C3 python tools/plan_time.py > /dev/null 2>&1
for rep in gpurun_out/${R}_*.ncu-rep; do
    [ -f "$rep" ] || continue
    b=$(basename "$rep" .ncu-rep)
    python tools/ncu_summary.py "$rep" > "gpurun_out/${b/${R}_/${R}_ncu_}.txt" 2>&1 && rm -f "$rep"
done
timeout 300 python tools/step_gaps.py C3 > gpurun_out/${R}_step_gaps.txt 2>&1
timeout 600 python tools/resmode_time.py C1 C2 C3 C4 C5 > gpurun_out/${R}_resmode_time.md 2>&1
timeout 300 python tools/loop_scan.py > gpurun_out/${R}_loop_scan_final.txt 2>&1
ls -la gpurun_out | grep ${R}

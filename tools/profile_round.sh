#!/bin/bash
# One GPU session of evidence for profiles/: plain bench, launch list of the same command,
# one ncu --set full capture of the loop kernel at C3 and C4 (capped) and of the sketch at C4.
# usage (under gpurun): bash tools/profile_round.sh r01
set -x
R=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench.log 2>&1 || exit 1
CSK_PROFILE_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-e2e \
    > gpurun_out/${R}_ncu_launches.log 2>&1
python tools/run_solve_once.py C3 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${R}_loop_C3 python tools/run_solve_once.py C3 > gpurun_out/${R}_ncu_loop_C3.log 2>&1
python tools/run_solve_once.py C4 2000 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${R}_loop_C4 python tools/run_solve_once.py C4 2000 > gpurun_out/${R}_ncu_loop_C4.log 2>&1
python tools/sketch_time.py C3 > /dev/null 2>&1 && \
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_dense -s 2 -c 1 \
    -o gpurun_out/${R}_sketch_C3 python tools/sketch_time.py C3 > gpurun_out/${R}_ncu_sketch_C3.log 2>&1
ls -la gpurun_out
# stream-ring loop (C5, capped) and the warp-per-bucket sketch (Table-1 shape)
python tools/run_c5_once.py 100 > /dev/null 2>&1 && \
CSK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_loop -c 1 \
    -o gpurun_out/${R}_loop_C5 python tools/run_c5_once.py 100 > gpurun_out/${R}_ncu_loop_C5.log 2>&1
python tools/csk_breakdown.py 700000x150 > /dev/null 2>&1 && \
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_dense_wpb -s 2 -c 1 \
    -o gpurun_out/${R}_sketch_wpb python tools/csk_breakdown.py 700000x150 > gpurun_out/${R}_ncu_sketch_wpb.log 2>&1
ls -la gpurun_out
# summarise on the box and drop the reports (gpurun merges at most 64 MiB of gpurun_out/)
for rep in gpurun_out/${R}_*.ncu-rep; do
    [ -f "$rep" ] || continue
    b=$(basename "$rep" .ncu-rep)
    python tools/ncu_summary.py "$rep" > "gpurun_out/${b/${R}_/${R}_ncu_}.txt" 2>&1 && rm -f "$rep"
done
ls -la gpurun_out

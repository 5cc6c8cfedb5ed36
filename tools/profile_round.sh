#!/bin/bash
# One GPU session of evidence for profiles/: pytest -m gpu, the plain bench line, the launch list
# of the same command (ncu --metrics gpu__time_duration.sum, cold-cache and serialised), and one
# ncu --set full capture each of the loop at C3 / C4 (capped), the dense sketch at C3 / C4, the
# CSR sketch at C5 and the plan at C5; summarised on the box (tools/ncu_summary.py), reports
# dropped (gpurun merges at most 64 MiB).      usage (under gpurun): bash tools/profile_round.sh r02
R=${1:-r02}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${R}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${R}_pytest_gpu.log
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
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_dense -s 2 -c 1 \
    -o gpurun_out/${R}_sketch_C4 python tools/sketch_time.py C4 > /dev/null 2>&1
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_csr -s 2 -c 1 \
    -o gpurun_out/${R}_sketch_csr_C5 python tools/csr_time.py 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plan_hist -s 37 -c 1 \
    -o gpurun_out/${R}_plan_C5 python tools/plan_time.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_row_norms_staged -s 2 -c 1 \
    -o gpurun_out/${R}_norms_C5 python tools/csr_time.py 3 > /dev/null 2>&1
# NVTX: only the kernels inside the csk_sketch / csk_solve_ex ranges are profiled (the ranges exist)
timeout 300 ncu --nvtx --nvtx-include "csk_sketch/" --nvtx-include "csk_solve_ex/" --metrics gpu__time_duration.sum \
    --csv python tools/run_solve_once.py C1 > gpurun_out/${R}_nvtx_ranges.csv 2>&1
# the random-gather floor of C5's CSR access pattern, the norms and CSR kernel times, Table 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu && \
    timeout 300 ./tools/microbench_gather > gpurun_out/${R}_microbench_gather.txt 2>&1
timeout 300 python tools/norms_time.py > gpurun_out/${R}_norms_time.txt 2>&1
timeout 300 python tools/csr_time.py 5 > gpurun_out/${R}_csr_time.txt 2>&1
timeout 1800 python tools/table1.py --trials 50 --json gpurun_out/${R}_table1.json > gpurun_out/${R}_table1.md 2>&1
for rep in gpurun_out/${R}_*.ncu-rep; do
    [ -f "$rep" ] || continue
    b=$(basename "$rep" .ncu-rep)
    python tools/ncu_summary.py "$rep" > "gpurun_out/${b/${R}_/${R}_ncu_}.txt" 2>&1 && rm -f "$rep"
done
timeout 600 python tools/resmode_time.py C1 C2 C3 C4 C5 > gpurun_out/${R}_resmode_time.md 2>&1
ls -la gpurun_out | grep ${R}

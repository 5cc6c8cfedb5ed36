#!/bin/bash
# The rest of profile_round.sh at the final build (Table 1, NVTX ranges, CSR / norms times, the
# gather floor, the CSR and norms ncu summaries): usage (under gpurun): bash tools/gpu_final2.sh r02z
R=${1:-r02z}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_csr -s 2 -c 1 \
    -o gpurun_out/${R}_sketch_csr_C5 python tools/csr_time.py 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_row_norms_staged -s 2 -c 1 \
    -o gpurun_out/${R}_norms_C5 python tools/csr_time.py 3 > /dev/null 2>&1
for rep in gpurun_out/${R}_*.ncu-rep; do
    [ -f "$rep" ] || continue
    b=$(basename "$rep" .ncu-rep)
    python tools/ncu_summary.py "$rep" > "gpurun_out/${b/${R}_/${R}_ncu_}.txt" 2>&1 && rm -f "$rep"
done
timeout 300 ncu --nvtx --nvtx-include "csk_sketch/" --nvtx-include "csk_solve_ex/" --metrics gpu__time_duration.sum \
    --csv python tools/run_solve_once.py C1 > gpurun_out/${R}_nvtx_ranges.csv 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu && \
    timeout 300 ./tools/microbench_gather > gpurun_out/${R}_microbench_gather.txt 2>&1
timeout 300 python tools/norms_time.py > gpurun_out/${R}_norms_time.txt 2>&1
timeout 300 python tools/csr_time.py 5 > gpurun_out/${R}_csr_time.txt 2>&1
timeout 2400 python tools/table1.py --trials 50 --json gpurun_out/${R}_table1.json > gpurun_out/${R}_table1.md 2>&1
ls -la gpurun_out | grep ${R}

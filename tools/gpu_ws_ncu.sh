cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-wsn}
CSK_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(plan|hash|sketch|row|offsets|scan|hist|count|bucket)' -s 6 -c 12 --csv python tools/csr_time.py 3 > gpurun_out/${T}_csr_launches.csv 2>&1
CSK_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_csr -s 1 -c 1 -o gpurun_out/${T}_csr python tools/csr_time.py 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_csr.ncu-rep > gpurun_out/${T}_ncu_csr.txt 2>&1

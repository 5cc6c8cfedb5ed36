cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for spec in "ab/libcsk_pl.so"; do
  echo "== $spec" >> gpurun_out/${TAG}_plan_k.txt
  bash tools/plan_kernel_time.sh $spec >> gpurun_out/${TAG}_plan_k.txt 2>&1
done
CSK_LIB=$PWD/ab/libcsk_pl.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plan_hist -s 14 -c 1 -o gpurun_out/${TAG}_plan_C3 python tools/plan_time.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_plan_C3.ncu-rep > gpurun_out/${TAG}_ncu_plan_C3.txt 2>&1 && rm -f gpurun_out/${TAG}_plan_C3.ncu-rep

#!/bin/bash
# DRAM bytes and L2 hit rate of k_loop at C5 (100 iterations) without and with the L2-resident
# streamed rows.  usage (under gpurun): bash tools/gpu_l2pin_ncu.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/run_c5_once.py 100 > gpurun_out/r02_c5_once.log 2>&1 || exit 1
for mb in 0 96; do
  CSK_PROFILE_NONCOOP=1 CSK_LOOP_L2PIN_MB=$mb timeout 900 ncu \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_loop -c 1 --csv --log-file gpurun_out/r02_ncu_c5_l2pin_$mb.csv \
    python tools/run_c5_once.py 100 > /dev/null 2>&1
  echo "== CSK_LOOP_L2PIN_MB=$mb"; grep -v "^==" gpurun_out/r02_ncu_c5_l2pin_$mb.csv | cut -d, -f5,13- | tail -6
done

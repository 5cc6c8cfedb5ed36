# kernel time of k_plan_hist per size (ncu gpu__time_duration, cold and serialised): bash tools/plan_kernel_time.sh <lib> [env...]
L=$1; shift
env "$@" CSK_LIB=$PWD/$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_plan_hist --csv python tools/plan_time.py 2>/dev/null | grep k_plan_hist | awk -F'","' '{print $NF}' | tr -d '"' | paste -sd' ' | awk '{for(i=1;i<=NF;i+=6){s="";for(j=i+1;j<i+6;j++)s=s" "$j; print s}}'

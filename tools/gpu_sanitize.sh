cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for part in plan sketch loop sharded; do
    echo "=== $tool $part" >> gpurun_out/${TAG}_sanitize.txt
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py $part >> gpurun_out/${TAG}_sanitize.txt 2>&1
    echo "exit $?" >> gpurun_out/${TAG}_sanitize.txt
  done
done

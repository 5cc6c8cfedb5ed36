cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "exit $?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>> gpurun_out/${TAG}_bench.err
timeout 600 python tools/distortion.py C1 C2 C3 300000x50 300000x100 > gpurun_out/${TAG}_distortion.md 2>&1

cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --sharded --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_sharded.json 2> gpurun_out/${TAG}_bench_sharded.err
tail -3 gpurun_out/${TAG}_pytest.log

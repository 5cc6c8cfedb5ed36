#!/bin/bash
# A/B of the speculative winner copies (CSK_SPEC_ROW=1 build, libcsk_spec.so) against the product
# build: parity tests through the spec build, loop us/iteration per config, the C3 bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CSK_LIB=$PWD/paper_2004_02480_b200/libcsk_spec.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "C3_full or small_configs or launch_shapes or residual or warm_start or edge_cases or stream_ring or mwrk or run_and_run_host" \
  > gpurun_out/spec_pytest.log 2>&1; echo "exit $?" >> gpurun_out/spec_pytest.log
timeout 900 python tools/loop_ab.py paper_2004_02480_b200/libcsk.so paper_2004_02480_b200/libcsk_spec.so \
  paper_2004_02480_b200/libcsk.so paper_2004_02480_b200/libcsk_spec.so --configs=C1,C3,C4 > gpurun_out/spec_ab.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-extras --no-cpu --no-e2e > gpurun_out/spec_bench_base.json 2>/dev/null
CSK_LIB=$PWD/paper_2004_02480_b200/libcsk_spec.so timeout 600 python bench.py --steps 20 --warmup 3 --no-extras --no-cpu --no-e2e > gpurun_out/spec_bench_spec.json 2>/dev/null
tail -3 gpurun_out/spec_pytest.log; cat gpurun_out/spec_ab.txt
for f in base spec; do python -c "import json,sys;d=json.loads(open('gpurun_out/spec_bench_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['us_per_iteration'],d['iterations'])"; done

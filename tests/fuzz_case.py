"""Re-run one fuzz case with option variants: python tests/fuzz_case.py m n d kind seed"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, paper_2004_02480_b200 as csk
from csk_synth import make_dense
from test_gpu_parity import _lockstep, _np
m, n, d, kind, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
p = make_dense(m, n, kind, 7000 + k, "cuda")
At, bt, nsq = csk.csk_sketch(p.A, p.b, d, seed=k)
for opts in [{}, {"smem_rows": -1}, {"cluster_size": 1, "num_ctas": 148}, {"num_ctas": 100}, {"reg_rows": 8}]:
    try:
        g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=1e-30, max_iters=40, trace=41, trace_x=True, **opts)
        try:
            _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 40)
            res = "ok"
        except AssertionError as e:
            res = f"FAIL {e}"
        print(opts, csk.csk_last_solve_tiers(), res, flush=True)
    except Exception as e:
        print(opts, "error", e, flush=True)

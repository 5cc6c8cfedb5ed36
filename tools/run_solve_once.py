"""Run one sketch + one solve of a config (for ncu captures of the loop kernel).

python tools/run_solve_once.py C3 [max_iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

nm = sys.argv[1] if len(sys.argv) > 1 else "C3"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = CONFIGS[nm]
p = make_config(cfg, "cuda")
At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
r = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=cfg.tol, max_iters=cap or cfg.max_iters)
torch.cuda.synchronize()
print(nm, "IT", r.iterations, "RES", r.final_res, "term", r.termination)

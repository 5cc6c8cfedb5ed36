"""One C5 solve capped at N iterations (for ncu -k regex:k_loop): python tools/run_c5_once.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfg = CONFIGS["C5"]
p = make_config(cfg, "cuda")
At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, p.n, cfg.d, seed=cfg.sketch_seed)
r = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap)
torch.cuda.synchronize()
print("C5", r.iterations, r.final_res, csk.csk_last_solve_tiers())

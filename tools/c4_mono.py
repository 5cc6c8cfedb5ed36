"""Debug: C4 RES monotonicity and where two libs' trajectories part (CSK_LIB picks the .so)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_02480_b200 as csk
from csk_synth import CONFIGS, make_config
cfg = CONFIGS["C4"]
p = make_config(cfg, "cuda")
At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
cap = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, trace=cap + 1)
res = g.res_trace.cpu().numpy()
idx = g.idx_trace.cpu().numpy()
bad = np.nonzero(np.diff(res) > 1e-12 * res[:-1])[0]
print(os.path.basename(csk.LIB_PATH), "IT", g.iterations, "violations", len(bad), bad[:10], res[bad[:3]], res[bad[:3] + 1])
np.save(os.path.join("gpurun_out", "c4_idx_" + os.path.basename(csk.LIB_PATH) + ".npy"), idx)

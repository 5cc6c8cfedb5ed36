"""Loop time per iteration vs CTA count: python tools/ctas_sweep.py C3 148 120 100 74"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2004_02480_b200 as csk
from csk_synth import CONFIGS, make_config
nm = sys.argv[1]
cfg = CONFIGS[nm]
p = make_config(cfg, "cuda")
At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
for G in [int(v) for v in sys.argv[2:]]:
    best = 1e30
    for _ in range(3):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        r = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=3000, num_ctas=G, cluster_size=1)
        en.record()
        torch.cuda.synchronize()
        best = min(best, st.elapsed_time(en))
    print(f"{nm} ctas={G} IT={r.iterations} {best * 1e3 / r.iterations:.3f} us/iter {csk.csk_last_solve_tiers()}", flush=True)

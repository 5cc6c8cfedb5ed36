"""Cluster vs grid exchange per config: python tools/cluster_ab.py C1 C2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

for nm in [a for a in sys.argv[1:] if a in CONFIGS]:
    cfg = CONFIGS[nm]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
    for cs, nc in [(0, 0), (16, 0), (1, 0), (1, 64), (1, 32)]:
        best = 1e30
        for _ in range(4):
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st.record()
            r = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=3000, cluster_size=cs, num_ctas=nc)
            en.record()
            torch.cuda.synchronize()
            best = min(best, st.elapsed_time(en))
        print(f"{nm} cluster={cs} ctas={nc} IT={r.iterations} {best * 1e3 / r.iterations:.3f} us/iter "
              f"{csk.csk_last_solve_tiers()}", flush=True)

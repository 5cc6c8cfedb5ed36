"""A/B timing of the loop kernel: python tools/ab_solve.py C3 [reps]  (uses CSK_LIB to pick the .so)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

names = [a for a in sys.argv[1:] if a in CONFIGS] or ["C3"]
for nm in names:
    cfg = CONFIGS[nm]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
    cap = cfg.max_iters if nm != "C4" else 5000
    best = 1e30
    for _ in range(5):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        r = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=cfg.tol, max_iters=cap)
        en.record()
        torch.cuda.synchronize()
        best = min(best, st.elapsed_time(en))
    print(f"{os.path.basename(csk.LIB_PATH)} {nm} IT={r.iterations} {best * 1e3 / r.iterations:.3f} us/iter "
          f"({best:.3f} ms)", flush=True)

"""MWRK on the unsketched system (Remark 1): the loop kernel on
(A, b, ||A_i||^2) with A streamed from L2/HBM every iteration.
python tools/mwrk_time.py C2 C3 [cap]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

cap = int(next((a for a in sys.argv[1:] if a.isdigit()), "200"))
for nm in [a for a in sys.argv[1:] if a in CONFIGS]:
    cfg = CONFIGS[nm]
    p = make_config(cfg, "cuda")
    nsq = csk.csk_row_norms(p.A)
    for rep in range(3):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        r = csk.csk_solve(p.A, p.b, nsq, x_star=p.x_star, tol=cfg.tol, max_iters=cap)
        en.record()
        torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    geo = csk.csk_last_solve_geometry()
    gbs = cfg.m * cfg.n * 8 * r.iterations / (ms * 1e-3) / 1e9
    print(f"{nm} MWRK m={cfg.m} n={cfg.n} IT={r.iterations} ({r.termination}) {ms:.2f} ms "
          f"{ms * 1e3 / r.iterations:.2f} us/iter {gbs:.0f} GB/s geo={geo}", flush=True)

"""Loop time per iteration where rows are streamed from L2/HBM every iteration: C5 (CSR sketch,
A~ = 40000 x 2000 = 640 MB > on-chip) and MWRK on the unsketched C3 / Table-1 systems.
python tools/stream_time.py [cap]   (uses CSK_LIB to pick the .so)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

cap = int(next((a for a in sys.argv[1:] if a.isdigit()), "60"))
lib = os.path.basename(csk.LIB_PATH)


def timed(At, bt, nsq, xs, label, bytes_per_it):
    best = 1e30
    for _ in range(3):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        r = csk.csk_solve(At, bt, nsq, x_star=xs, max_iters=cap)
        en.record()
        torch.cuda.synchronize()
        best = min(best, st.elapsed_time(en))
    us = best * 1e3 / r.iterations
    print(f"{lib} {label} IT={r.iterations} {us:.2f} us/iter {bytes_per_it / (us * 1e-6) / 1e9:.0f} GB/s "
          f"(A bytes / iteration time) geo={csk.csk_last_solve_geometry()}", flush=True)


cfg = CONFIGS["C5"]
p = make_config(cfg, "cuda")
At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, p.n, cfg.d, seed=cfg.sketch_seed)
del p.row_ptr, p.col, p.val
timed(At, bt, nsq, p.x_star, "C5 CSK loop", 8 * cfg.d * cfg.n)
del At, bt, nsq
for (m, n) in [(700000, 50), (700000, 100), (700000, 150)]:
    g = torch.Generator(device="cuda").manual_seed(5)
    xs = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    timed(A, A @ xs, csk.csk_row_norms(A), xs, f"MWRK {m}x{n}", 8 * m * n)
cfg = CONFIGS["C3"]
p = make_config(cfg, "cuda")
timed(p.A, p.b, csk.csk_row_norms(p.A), p.x_star, "MWRK C3", 8 * cfg.m * cfg.n)

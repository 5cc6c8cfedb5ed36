"""Loop us/iteration vs rows per CTA and row length (what the exchange costs with no GEMV to speak of):
python tools/loop_scan.py   -- random A~ (d x n), b~ = A~ x*, 1500 iterations capped, best of 3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402


def one(d, n, cap=1500, **kw):
    g = torch.Generator(device="cuda").manual_seed(d * 7919 + n)
    At = torch.randn(d, n, dtype=torch.float64, device="cuda", generator=g)
    xs = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    bt = At @ xs
    nsq = (At * At).sum(1)
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = csk.csk_solve(At, bt, nsq, x_star=xs, tol=1e-30, max_iters=cap, **kw)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / max(r.iterations, 1))
    return best, csk.csk_last_solve_tiers()


for n in (500, 50, 1000):
    for d in (148, 296, 592, 1480, 2960, 5000, 10000):
        if n != 500 and d not in (148, 1480, 5000, 10000):
            continue
        t, tiers = one(d, n, cluster_size=1)
        print(f"n={n} d={d} rows/CTA={(d + 147) // 148}: {t:.3f} us/iter {tiers}", flush=True)

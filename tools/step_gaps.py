"""Where the C3 step's time goes outside the kernels: CUDA events between the public calls of one
step (plan / sketch on the plan / norms / solve) and the host time of each call.
python tools/step_gaps.py [config]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "C3"
if spec in CONFIGS:
    cfg = CONFIGS[spec]
    p = make_config(cfg, "cuda")
else:  # "MxN" (the paper's Table-1 shapes: d = n^2, Gaussian A, b = A x*)
    from types import SimpleNamespace
    m_, n_ = (int(v) for v in spec.split("x"))
    g = torch.Generator(device="cuda").manual_seed(m_ + n_)
    xs_ = torch.randn(n_, generator=g, device="cuda", dtype=torch.float64)
    A_ = torch.randn(m_, n_, generator=g, device="cuda", dtype=torch.float64)
    cfg = SimpleNamespace(name=spec, m=m_, n=n_, d=n_ * n_, sketch_seed=0, tol=1e-6, max_iters=20000)
    p = SimpleNamespace(A=A_, b=A_ @ xs_, x_star=xs_)
ctx = csk.Context()
csk.csk_ctx_set_timing(True, ctx=ctx)
d, n = cfg.d, cfg.n
At = torch.empty(d, n, dtype=torch.float64, device="cuda")
bt = torch.empty(d, dtype=torch.float64, device="cuda")
nsq = torch.empty(d, dtype=torch.float64, device="cuda")
x = torch.zeros(n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()


def whole(ev, ht):
    x.zero_()
    t0 = time.perf_counter()
    ev[0].record(s)
    csk.csk_sketch(p.A, p.b, d, seed=cfg.sketch_seed, ctx=ctx, out=(At, bt, nsq))
    ev[1].record(s)
    t1 = time.perf_counter()
    csk.csk_solve_async(At, bt, nsq, x, x_star=p.x_star, tol=cfg.tol, max_iters=cfg.max_iters, ctx=ctx)
    ev[2].record(s)
    t2 = time.perf_counter()
    r = csk.csk_solve_wait(ctx)
    ht.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6))
    return r


rows = {"sketch call": [], "solve call": [], "sketch kernel": [], "loop kernel": [], "host sketch": [],
        "host solve": []}
for k in range(12):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ht = []
    whole(ev, ht)
    torch.cuda.synchronize()
    if k < 3:
        continue
    rows["sketch call"].append(ev[0].elapsed_time(ev[1]) * 1e3)
    rows["solve call"].append(ev[1].elapsed_time(ev[2]) * 1e3)
    rows["sketch kernel"].append(csk.csk_last_kernel_ms("sketch", ctx=ctx) * 1e3)
    rows["loop kernel"].append(csk.csk_last_kernel_ms("loop", ctx=ctx) * 1e3)
    rows["host sketch"].append(ht[0][0])
    rows["host solve"].append(ht[0][1])
for k, v in rows.items():
    print(f"{cfg.name} {k:14s} median {statistics.median(v):9.1f} us  (min {min(v):.1f}, max {max(v):.1f})")
# the parts on their own (events around each public call)

for name, fn in [("plan", lambda: csk.csk_plan(cfg.m, d, seed=cfg.sketch_seed, ctx=ctx)),
                 ("norms", lambda: csk.csk_row_norms(At, ctx=ctx))]:
    ts = []
    for k in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        if k >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    print(f"{cfg.name} {name:14s} alone  {statistics.median(ts):9.1f} us")

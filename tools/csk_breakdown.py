"""Where the time of one CSK run goes (Table-1 sizes): whole csk_sketch call, the sketch kernel
alone, whole csk_solve call, the loop kernel alone (libcsk kernel events).
python tools/csk_breakdown.py 300000x50 700000x150"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402

ctx = csk.Context()
csk.csk_ctx_set_timing(True, ctx=ctx)
for spec in sys.argv[1:]:
    m, n = (int(v) for v in spec.split("x"))
    d = n * n
    g = torch.Generator(device="cuda").manual_seed(3)
    xs = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    b = A @ xs
    At = torch.empty(d, n, dtype=torch.float64, device="cuda")
    bt = torch.empty(d, dtype=torch.float64, device="cuda")
    nsq = torch.empty(d, dtype=torch.float64, device="cuda")
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    for seed in (0, 0, 0, 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        x.zero_()
        ev[0].record()
        csk.csk_sketch(A, b, d, seed=seed, ctx=ctx, out=(At, bt, nsq))
        ev[1].record()
        csk.csk_solve_async(At, bt, nsq, x, x_star=xs, max_iters=20000, ctx=ctx)
        ev[2].record()
        r = csk.csk_solve_wait(ctx)
        torch.cuda.synchronize()
        print(f"{m}x{n} d={d} seed={seed}: sketch call {ev[0].elapsed_time(ev[1]):.3f} ms (kernel "
              f"{csk.csk_last_kernel_ms('sketch', ctx=ctx):.3f}), solve call {ev[1].elapsed_time(ev[2]):.3f} ms "
              f"(loop kernel {csk.csk_last_kernel_ms('loop', ctx=ctx):.3f}, IT={r.iterations}, "
              f"{csk.csk_last_solve_tiers(ctx=ctx)})", flush=True)

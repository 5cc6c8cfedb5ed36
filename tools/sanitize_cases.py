"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) covering every
kernel family: the plan (k_plan_fused, explicit map), the three sketch kernels, exact row norms,
the persistent loop (16-CTA cluster, grid exchange, TMEM tier, stream ring, residual stop), the
virtual-rank SYS loop and the CSR row routing.  Checks results against each other, prints OK.

compute-sanitizer --tool memcheck python tools/sanitize_cases.py [subset]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CSK_EXCHANGE_TIMEOUT_S", "900")
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import make_csr, make_dense  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(name, fn):
    if which not in ("all", name):
        return
    fn()
    torch.cuda.synchronize()
    print(f"{name}: OK", flush=True)


def plan():
    perm, offs = csk.csk_plan(20000, 2000, seed=3)
    h = torch.arange(3000, dtype=torch.int32, device="cuda") % 700
    s = torch.ones(3000, dtype=torch.int8, device="cuda")
    csk.csk_plan(3000, 700, h=h, sign=s)


def sketch():
    for m, n, d in [(6000, 40, 500), (6000, 300, 400)]:  # warp-per-bucket, TMA ring
        p = make_dense(m, n, "gauss", 1, "cuda")
        At, bt, nsq = csk.csk_sketch(p.A, p.b, d, seed=2)
        assert torch.equal(nsq, csk.csk_row_norms(At))
    p = make_csr(4000, 300, 8, seed=2, device="cuda")
    csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, 300, 350, seed=1)


def loop():
    p = make_dense(1000, 50, "gauss", 1000, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, 500, seed=0)
    for cs in (16, 1):  # the 16-CTA cluster exchange, the grid-wide atomic exchange
        g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, cluster_size=cs, max_iters=60, tol=1e-30)
        assert g.iterations == 60
    csk.csk_solve(At, bt, nsq, x_star=None, cluster_size=1, max_iters=40, tol=1e-30)  # residual stop
    p = make_dense(4000, 200, "gauss", 5, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, 1500, seed=5)
    csk.csk_solve(At, bt, nsq, x_star=p.x_star, num_ctas=12, tmem=True, max_iters=30, tol=1e-30)  # TMEM tier
    csk.csk_solve(At, bt, nsq, x_star=p.x_star, num_ctas=4, max_iters=30, tol=1e-30)  # stream ring


def sharded():
    p = make_dense(1000, 50, "gauss", 1000, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, 500, seed=0)
    csk.csk_solve_virtual_ranks(At, bt, nsq, 2, x_star=p.x_star, max_iters=40, tol=1e-30)
    q = make_csr(3000, 64, 6, seed=4, device="cuda")
    csk.csk_sketch_csr_routed_virtual(q.row_ptr, q.col, q.val, q.b, 64, 200, 2, seed=1)


run("plan", plan)
run("sketch", sketch)
run("loop", loop)
run("sharded", sharded)

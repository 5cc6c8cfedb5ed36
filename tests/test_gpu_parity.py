"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE north_star):
  * h, D, perm, offsets, A~, b~: bit-exact at P = 1 (the sketch is a fixed-order
    fold of exactly representable +-A values);
  * nsq: bit-exact too (S4 runs the oracle's left-to-right fma chain, one thread per row);
  * loop: lockstep -- given the GPU's x_k, the GPU's residual vector r_k (traced by the kernel's
    finalize, csk_solve_opts_t.r_trace) is within 1e-10 of the oracle's r(x_k) in the 2-norm,
    relative (north_star); the oracle's scores (its own row norms) pick the same i_k (or a
    near-tie within 4e-10 relative); the oracle's step from (x_k, i_k) lands on the GPU's
    x_{k+1} within 1e-12 relative; free-running -- RES <= tol for both and
    |IT_gpu - IT_orc| <= max(1, 5 % IT_orc).
"""
import numpy as np
import pytest
import torch

import oracle
from csk_synth import CONFIGS, make_config, make_dense

pytestmark = pytest.mark.gpu

U = 2.0**-53


@pytest.fixture(scope="module")
def csk():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2004_02480_b200 as m
    return m


def _np(t):
    return t.detach().cpu().numpy()


def _check_sketch(csk, A, b, d, seed, **kw):
    At, bt, nsq = csk.csk_sketch(A, b, d, seed=seed, **kw)
    torch.cuda.synchronize()
    An = _np(A)
    At_o, bt_o = oracle.sketch_dense(An, _np(b), d, seed=seed)
    assert np.array_equal(_np(At), At_o), "A~ not bit-exact"
    assert np.array_equal(_np(bt), bt_o), "b~ not bit-exact"
    nsq_o = oracle.row_norms(At_o)
    assert np.array_equal(_np(nsq), nsq_o), "nsq not bit-exact (S4 in the oracle's fma order)"
    nsq2 = csk.csk_row_norms(At)
    assert torch.equal(nsq, nsq2), "sketch and standalone row norms differ"
    return At, bt, nsq


@pytest.mark.parametrize("d,n,offset", [(1, 2, 0), (31, 64, 0), (33, 130, 0), (70, 500, 0), (100, 2000, 0),
                                        (65, 63, 0), (40, 7, 0), (50, 500, 1), (5, 1, 0), (3, 66, 0)])
def test_row_norms_paths(csk, d, n, offset):
    """S4 bit-exact on both norm kernels: the TMA-staged one (n even, 16-byte aligned rows: full
    and partial 64-column stages, d not a multiple of 32) and the plain one (odd n, or A~ starting
    8 bytes off a 16-byte boundary)."""
    g = torch.Generator().manual_seed(d * 1000 + n)
    flat = torch.randn(d * n + offset, generator=g, dtype=torch.float64)
    A = flat[offset:].view(d, n)
    nsq = csk.csk_row_norms(A.cuda()[0:d] if offset == 0 else flat.cuda()[offset:].view(d, n))
    assert np.array_equal(_np(nsq), oracle.row_norms(A.numpy()))


# ---------------------------------------------------------------- S1/S2
@pytest.mark.parametrize("seed,m,d,off", [(0, 1000, 500, 0), (0, 20000, 2000, 0),
                                          (2**63 + 5, 123457, 40000, 0), (7, 5000, 3, 1234)])
def test_hash_bitexact(csk, seed, m, d, off):
    h, s = csk.csk_hash(m, d, seed=seed, row_offset=off)
    ho, so = oracle.hash_map(seed, m + off, d)
    assert np.array_equal(_np(h), ho[off:])
    assert np.array_equal(_np(s), so[off:])


@pytest.mark.parametrize("m,d", [(1000, 500), (100000, 5000), (77777, 1), (4096, 4095), (20000, 2000),
                                 (60000, 400), (199999, 40000), (8193, 8000), (150000, 70000), (300000, 1000),
                                 (5, 2)])
def test_plan_bitexact(csk, m, d):
    """Every plan path gives the oracle's stable bucketing (plan.cu): the histogram plan (d counts in
    shared memory; groups of one CTA sharing a bucket sorted), the global-atomic plan with the warp
    bitonic sort (d = 70000 > shared memory), the CUB radix sort (m > 512 d: d = 1)."""
    perm, offs = csk.csk_plan(m, d, seed=11)
    h, s = oracle.hash_map(11, m, d)
    order = np.argsort(h, kind="stable")
    want = order.astype(np.int64) | np.where(s[order] < 0, 1 << 31, 0)
    got = _np(perm).astype(np.int64) & 0xFFFFFFFF
    assert np.array_equal(got, want)
    assert np.array_equal(_np(offs), np.searchsorted(h[order], np.arange(d + 1), side="left"))


@pytest.mark.parametrize("m,d,pattern", [(227328, 500, "mod32"), (227328, 500, "mod500"),
                                         (150000, 3000, "runs"), (100000, 5000, "reverse")])
def test_plan_explicit_map_collisions(csk, m, d, pattern):
    """Explicit maps built to collide inside the histogram plan's 512-row chunks: h = i mod 32
    (every warp of every chunk claims the same 32 buckets, so the list of colliding groups
    overflows and the plan sorts every group), i mod d, runs of equal buckets and a descending
    map -- the stable order (rows ascending inside a bucket) in every case."""
    i = np.arange(m, dtype=np.int64)
    h = {"mod32": i % 32, "mod500": i % d, "runs": (i // 37) % d, "reverse": (d - 1) - (i * d) // m}[pattern]
    h = h.astype(np.int32)
    s = np.where((i * 2654435761) % 7 < 3, -1, 1).astype(np.int8)
    perm, offs = csk.csk_plan(m, d, h=torch.from_numpy(h).cuda(), sign=torch.from_numpy(s).cuda())
    order = np.argsort(h, kind="stable")
    want = order.astype(np.int64) | np.where(s[order] < 0, 1 << 31, 0)
    got = _np(perm).astype(np.int64) & 0xFFFFFFFF
    assert np.array_equal(got, want)
    assert np.array_equal(_np(offs), np.searchsorted(h[order], np.arange(d + 1), side="left"))


# ---------------------------------------------------------------- S3/S4
@pytest.mark.parametrize("m,n,d", [(1000, 50, 500), (20000, 200, 2000), (3001, 17, 700),
                                   (999, 1, 10), (4000, 2500, 300), (5000, 64, 4999),
                                   (2000, 333, 1), (6000, 1000, 100)])
def test_sketch_bitexact_shapes(csk, m, n, d):
    p = make_dense(m, n, "lognormal_rows", 77, "cuda")
    _check_sketch(csk, p.A, p.b, d, seed=3)


@pytest.mark.parametrize("n", [1, 2, 3, 63, 64, 65, 127, 128, 129, 255, 256, 257])
def test_sketch_short_row_boundaries(csk, n):
    """The warp-per-bucket kernel's column blocks (V = ceil(n/64) pairs per lane, odd tails) and
    its hand-over to the TMA ring kernel at n = 257; m = 20000 takes the one-launch plan."""
    p = make_dense(20000, n, "lognormal_rows", 500 + n, "cuda")
    _check_sketch(csk, p.A, p.b, 1000, seed=6)


@pytest.mark.parametrize("n,lda", [(50, 51), (64, 67), (200, 203)])
def test_sketch_short_rows_unaligned(csk, n, lda):
    """Odd lda (8-byte aligned rows): the warp-per-bucket kernel's scalar-load path."""
    p = make_dense(7000, n, "gauss", n + lda, "cuda")
    buf = torch.zeros(7000 * lda, dtype=torch.float64, device="cuda")
    Ab = buf.view(7000, lda)
    Ab[:, :n] = p.A
    At, bt, _ = csk.csk_sketch(Ab[:, :n], p.b, 600, seed=12)
    At_o, bt_o = oracle.sketch_dense(_np(p.A), _np(p.b), 600, seed=12)
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)


@pytest.mark.parametrize("m,n,lda,d", [(3000, 513, 514, 400), (2500, 777, 780, 300), (4000, 1000, 1000, 1999),
                                       (1500, 300, 300, 100), (2000, 2600, 2600, 64)])
def test_sketch_long_rows_padded(csk, m, n, lda, d):
    """Long rows through the TMA ring kernel: odd n (the last column read past the bulk copy),
    padded lda, a short last stage, several column chunks (n = 2600)."""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    buf = torch.randn(m * lda, generator=g, dtype=torch.float64, device="cuda")
    A = buf.view(m, lda)[:, :n]
    b = torch.randn(m, generator=g, dtype=torch.float64, device="cuda")
    At, bt, nsq = csk.csk_sketch(A, b, d, seed=21)
    At_o, bt_o = oracle.sketch_dense(_np(A.contiguous()), _np(b), d, seed=21)
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
    assert np.array_equal(_np(nsq), oracle.row_norms(At_o))


@pytest.mark.parametrize("lda,shift", [(136, 0), (131, 0), (130, 1)])
def test_sketch_padded_and_unaligned_lda(csk, lda, shift):
    """lda > n (even: TMA path), odd lda and an 8-byte-aligned A (plain-load path)."""
    p = make_dense(3000, 130, "gauss", 5, "cuda")
    buf = torch.zeros(3000 * lda + 8, dtype=torch.float64, device="cuda")
    Ab = buf[shift:shift + 3000 * lda].view(3000, lda)
    Ab[:, :130] = p.A
    At, bt, _ = csk.csk_sketch(Ab[:, :130], p.b, 400, seed=9)
    At_o, bt_o = oracle.sketch_dense(_np(p.A), _np(p.b), 400, seed=9)
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)


def test_sketch_identity_map_signed_rows(csk):
    """Remark 1: h = identity, d = m -> A~ = D A exactly."""
    p = make_dense(500, 40, "gauss", 8, "cuda")
    h = torch.arange(500, dtype=torch.int32, device="cuda")
    s = (torch.randint(0, 2, (500,), device="cuda", dtype=torch.int8) * 2 - 1).to(torch.int8)
    At, bt, _ = csk.csk_sketch_with_map(p.A, p.b, 500, h, s)
    sd = s.to(torch.float64)
    assert torch.equal(At, p.A * sd[:, None]) and torch.equal(bt, p.b * sd)


def test_sketch_argument_errors(csk):
    p = make_dense(100, 8, "gauss", 1, "cuda")
    with pytest.raises(csk.CskError) as e:
        csk.csk_sketch(p.A, p.b, 100)           # d == m violates d < m
    assert e.value.status == csk.CSK_E_ARG
    with pytest.raises(csk.CskError):
        csk.csk_sketch(p.A, p.b, 0)
    with pytest.raises(TypeError):              # no CPU fallback
        csk.csk_sketch(p.A.cpu(), p.b.cpu(), 10)


def test_sketch_with_cached_plan(csk):
    """csk_sketch_planned with a plan from csk_plan (computed once, reused): bit-exact."""
    p = make_dense(30000, 120, "lognormal_rows", 3, "cuda")
    perm, offs = csk.csk_plan(30000, 900, seed=8)
    for _ in range(2):
        At, bt, nsq = csk.csk_sketch_planned(p.A, p.b, 900, perm, offs)
        At_o, bt_o = oracle.sketch_dense(_np(p.A), _np(p.b), 900, seed=8)
        assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
        assert np.array_equal(_np(nsq), oracle.row_norms(At_o))


@pytest.mark.parametrize("timing", [False, True])
def test_sketch_graph_replay(csk, timing):
    """Repeated identical csk_sketch calls replay a captured CUDA graph (api.cu): every replay is
    bit-exact, a grown workspace re-captures, and with timing on the kernel events are recorded
    inside the graph (csk_last_kernel_ms of a replay is a real duration)."""
    ctx = csk.Context()
    if timing:
        csk.csk_ctx_set_timing(True, ctx=ctx)
    for m, n, d in [(3000, 64, 500), (3000, 64, 500), (3000, 64, 500), (9000, 96, 800), (9000, 96, 800),
                    (9000, 96, 800), (3000, 64, 500)]:
        p = make_dense(m, n, "gauss", m + n, "cuda")
        out = (torch.full((d, n), float("nan"), dtype=torch.float64, device="cuda"),
               torch.full((d,), float("nan"), dtype=torch.float64, device="cuda"),
               torch.full((d,), float("nan"), dtype=torch.float64, device="cuda"))
        for _ in range(4):  # eager, capture, replay, replay
            At, bt, _ = csk.csk_sketch(p.A, p.b, d, seed=4, ctx=ctx, out=out)
            torch.cuda.synchronize()
            At_o, bt_o = oracle.sketch_dense(_np(p.A), _np(p.b), d, seed=4)
            assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
            if timing:
                assert csk.csk_last_kernel_ms("sketch", ctx=ctx) > 0.0
            out[0].fill_(float("nan"))


# ---------------------------------------------------------------- S5-S8 loop
R_TOL = 1e-10  # north_star: per-iteration residuals within 1e-10 relative given the same x_k


def _check_r(r_gpu, r_orc, k, E=None):
    """||r_gpu - r_orc||_2 <= 1e-10 ||r_orc||_2 (normwise: elementwise relative error is unbounded
    where r_i ~ 0, e.g. at i_{k-1} right after its projection; SURVEY.md §8(c) acceptance 3) -- or,
    once the residual has shrunk to where fp64 cancellation decides (reading R-16), within the
    rounding bound of the two evaluations, ||E||_2 with E_i = 2 (n + 2) u (|b~_i| + sum_j |A~_ij x_j|):
    the exact r(x_k) itself is only known to that accuracy from any fp64 evaluation order."""
    err = float(np.linalg.norm(r_gpu - r_orc))
    bar = R_TOL * float(np.linalg.norm(r_orc))
    if E is not None:
        bar = max(bar, float(np.linalg.norm(E)))
    assert err <= bar, (k, err, float(np.linalg.norm(r_orc)), bar)


def _lockstep(At, bt, nsq, xtr, itr, k_max, rtr=None):
    """Step-for-step check of the GPU trajectory against the oracle.  Scores use the ORACLE's row
    norms (``nsq`` is accepted for the call sites' symmetry but not used), so a wrong GPU nsq
    cannot hide; ``rtr`` (the kernel's r_k trace) is checked against the oracle's r(x_k)."""
    At, bt = _np(At), _np(bt)
    nsq = oracle.row_norms(At)
    xtr, itr = _np(xtr), _np(itr)
    rtr = None if rtr is None else _np(rtr)
    if rtr is not None:
        assert len(rtr) >= min(k_max, len(itr)), "r trace shorter than the checked window"
    for k in range(min(k_max, len(itr), len(xtr) - 1)):
        r = oracle.residual(At, bt, xtr[k])
        if rtr is not None:
            E = 2 * (At.shape[1] + 2) * 2.0**-53 * (np.abs(bt) + np.abs(At) @ np.abs(xtr[k]))
            _check_r(rtr[k], r, k, E)
        mask = nsq > 0
        sc = np.where(mask, r * r / np.where(mask, nsq, 1), -1.0)
        io = int(np.argmax(sc))
        ig = int(itr[k])
        if ig != io and not sc[ig] >= (1 - 4e-10) * sc[io]:
            # a near-tie within rounding: both sides compute r_i = b~_i - A~_i x in fp64 in different
            # orders, |r_gpu - r_oracle| <= 2 (n+2) u (|b~_i| + sum_j |A~_ij x_j|) (R-10); once x_k is
            # near x* the residuals are that small (cancellation), and any row whose score can be
            # the largest within those bounds is a valid argmax
            n = At.shape[1]
            E = 2 * (n + 2) * 2.0**-53 * (np.abs(bt[[ig, io]]) + np.abs(At[[ig, io]]) @ np.abs(xtr[k]))
            hi_g = (abs(r[ig]) + E[0]) ** 2 / nsq[ig]
            lo_o = max(abs(r[io]) - E[1], 0.0) ** 2 / nsq[io]
            assert hi_g >= (1 - 4e-10) * lo_o, (k, ig, io, sc[ig], sc[io], E)
        lam = r[ig] / nsq[ig]
        x1 = xtr[k] + lam * At[ig]
        assert np.linalg.norm(x1 - xtr[k + 1]) <= 1e-12 * max(np.linalg.norm(x1), 1e-300) + 1e-14 * np.linalg.norm(lam * At[ig]), k


def _free_running(res_g, res_o):
    assert res_g.final_res <= 1e-6 and res_o.final_res <= 1e-6
    assert abs(res_g.iterations - res_o.iterations) <= max(1, 0.05 * res_o.iterations)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_solve_parity_small_configs(csk, name):
    cfg = CONFIGS[name]
    p = make_config(cfg, "cuda")
    At, bt, nsq = _check_sketch(csk, p.A, p.b, cfg.d, cfg.sketch_seed)
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=cfg.tol, max_iters=cfg.max_iters,
                      trace=4000, trace_x=True, trace_r=4000)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star),
                     tol=cfg.tol, max_iters=cfg.max_iters, trace=4000)
    assert g.termination == csk.CONVERGED
    _free_running(g, o)
    # every iteration, including the residual at the returned iterate (IT + 1 vectors)
    assert len(g.r_trace) == g.iterations + 1
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 4000, g.r_trace)
    Atn, btn, xn = _np(At), _np(bt), _np(g.x)
    E = 2 * (cfg.n + 2) * 2.0**-53 * (np.abs(btn) + np.abs(Atn) @ np.abs(xn))
    _check_r(_np(g.r_trace)[g.iterations], oracle.residual(Atn, btn, xn), g.iterations, E)
    n_same = min(len(g.idx_trace), len(o.idx_trace))
    assert np.array_equal(_np(g.idx_trace)[:n_same], o.idx_trace[:n_same])
    assert abs(g.final_res - oracle.solve(_np(At), _np(bt), _np(nsq), x0=_np(g.x), x_star=_np(p.x_star), max_iters=0).final_res) <= 1e-12


@pytest.mark.parametrize("num_ctas,smem_rows,cluster", [
    (1, 0, 1), (7, 0, 1), (148, -1, 1), (37, 40, 0), (2, -1, 2), (32, 0, 16), (112, -1, 16),
    (64, 17, 4), (16, 0, 8), (0, 0, 0), (146, 5, 2)])
def test_solve_launch_shapes_and_streamed_rows(csk, num_ctas, smem_rows, cluster):
    """Grids, cluster sizes (the DSMEM / global exchange hops) and the L2/HBM-streamed
    GEMV path (smem_rows = -1: no resident rows; k > 0: resident/streamed split)."""
    p = make_dense(8000, 300, "lognormal_rows", 91, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, 1500, seed=4)
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, num_ctas=num_ctas, smem_rows=smem_rows,
                      cluster_size=cluster, trace=300, trace_x=True, trace_r=300)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star), trace=300)
    _free_running(g, o)
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 300, g.r_trace)


@pytest.mark.parametrize("name,cluster,tmem", [("C1", 16, None), ("C1", 1, None), ("C2", 16, None),
                                               ("C2", 1, None), ("C2", 16, False), ("C2", 16, True)])
def test_solve_cluster_and_grid_exchange(csk, name, cluster, tmem):
    """The single-cluster DSMEM exchange (cluster_size=16) and the grid-wide atomic exchange
    (cluster_size=1) on the same sketched system: identical i_k sequences against the oracle."""
    cfg = CONFIGS[name]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=cfg.tol, max_iters=cfg.max_iters,
                      cluster_size=cluster, tmem=tmem, trace=4000, trace_x=True, trace_r=4000)
    geo = csk.csk_last_solve_geometry()
    assert geo["cluster_size"] == (16 if cluster == 16 else 1)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star),
                     tol=cfg.tol, max_iters=cfg.max_iters, trace=4000)
    assert g.termination == csk.CONVERGED
    _free_running(g, o)
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 4000, g.r_trace)
    n_same = min(len(g.idx_trace), len(o.idx_trace))
    assert np.array_equal(_np(g.idx_trace)[:n_same], o.idx_trace[:n_same])


@pytest.mark.parametrize("n,d,num_ctas,reg_rows,group_warps", [
    (200, 1500, 12, 0, 0),    # 8 register + 8 TMEM rows per group
    (200, 1500, 12, 2, 0),    # 2 register + 14 TMEM rows
    (201, 1600, 12, 0, 0),    # odd n: TMEM rows, plain-load row update
    (500, 3000, 10, 0, 0),    # all four tiers: registers, TMEM, shared memory, L2 stream
    (1000, 2400, 16, 3, 4),   # 4 warps per group (C4's layout), short register tier
    (2000, 3000, 20, 0, 8)])  # one 8-warp group per CTA (C5's per-GPU layout)
def test_solve_tmem_tier(csk, n, d, num_ctas, reg_rows, group_warps):
    """Rows of A~ held in tensor memory (tcgen05.st/ld, 8 columns per thread): same
    lockstep and free-running bars as the register/shared-memory tiers."""
    m = max(4 * d, 8 * n)
    p = make_dense(m, n, "gauss", 500 + n, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, d, seed=5)
    cap = 20000 if n <= 500 else 300
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, num_ctas=num_ctas, reg_rows=reg_rows,
                      group_warps=group_warps, tmem=True, trace=min(cap + 1, 400), trace_x=True, trace_r=150)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star), max_iters=cap,
                     trace=min(cap + 1, 400))
    if n <= 500:
        _free_running(g, o)
    else:
        assert g.termination == o.termination == csk.MAX_ITERS
        assert abs(g.final_res - o.final_res) <= 1e-6 * o.final_res
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 150, g.r_trace)
    n_same = min(len(g.idx_trace), len(o.idx_trace), 400)
    assert np.array_equal(_np(g.idx_trace)[:n_same], o.idx_trace[:n_same])


@pytest.mark.parametrize("n,rs", [(1000, 3), (1000, 5), (1000, 12), (999, 7)])
def test_solve_fused_tmem_smem_pass(csk, n, rs):
    """C4's layout (4 warps per group: 6 register rows, the full 16-row TMEM tier, rs shared-memory
    rows per thread) runs the interleaved TMEM + shared-memory pass (loop.cu tmem_smem_fused) with
    one 32-row tree: capped run with the oracle's i_k sequence and RES, lockstep with r_k."""
    G = 16
    d = G * 2 * (6 + 16 + rs)  # two 4-warp groups per CTA
    m = max(4 * d, 8 * n)
    p = make_dense(m, n, "gauss", 700 + n + rs, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, d, seed=rs)
    cap = 300
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, num_ctas=G, tmem=True, trace=cap + 1,
                      trace_x=True, trace_r=60)
    t = csk.csk_last_solve_tiers()
    assert (t["num_ctas"], t["group_warps"], t["reg_rows"], t["tmem_rows"], t["smem_rows"], t["ring_stages"]) == \
        (G, 4, 6, 16, rs, 0), t
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star), max_iters=cap,
                     trace=cap + 1)
    assert g.termination == o.termination == csk.MAX_ITERS
    assert np.array_equal(_np(g.idx_trace), o.idx_trace)
    assert abs(g.final_res - o.final_res) <= 1e-6 * o.final_res
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 60, g.r_trace)


@pytest.mark.parametrize("n", [1, 3, 63, 64, 65, 129, 1023, 2047, 2048])
def test_solve_ragged_n(csk, n):
    """Ragged widths around the 64-column lane groups and the n <= 2048 register limit.
    Small n: free-running parity to RES <= 1e-6.  Large n: a capped run (both stop at
    MaxIters) with the same i_k sequence and RES within 1e-6 relative, plus lockstep."""
    m = max(8 * n + 50, 400)
    d = max(4 * n, 50)
    p = make_dense(m, n, "gauss", 1000 + n, "cuda")
    At, bt, nsq = _check_sketch(csk, p.A, p.b, d, seed=n)
    cap = 20000 if n <= 129 else 150
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, trace=cap + 1, trace_x=n <= 129)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star),
                     max_iters=cap, trace=cap + 1)
    if n <= 129:
        _free_running(g, o)
        _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 50)
    else:
        assert g.termination == o.termination == csk.MAX_ITERS
        assert np.array_equal(_np(g.idx_trace), o.idx_trace)
        assert abs(g.final_res - o.final_res) <= 1e-6 * o.final_res
        g2 = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=8, tol=1e-30, trace=9, trace_x=True, trace_r=9)
        _lockstep(At, bt, nsq, g2.x_trace, g2.idx_trace, 8, g2.r_trace)


@pytest.mark.parametrize("num_ctas,cluster", [(0, 0), (148, 1), (64, 16)])
def test_solve_residual_mode(csk, num_ctas, cluster):
    p = make_dense(6000, 40, "gauss", 12, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, 400, seed=2)
    g = csk.csk_solve(At, bt, nsq, x_star=None, tol=1e-10, num_ctas=num_ctas, cluster_size=cluster)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=None, tol=1e-10)
    assert g.stop_mode == csk.STOP_RESIDUAL and g.termination == csk.CONVERGED
    assert abs(g.iterations - o.iterations) <= max(1, 0.05 * o.iterations)
    r = _np(bt) - _np(At) @ _np(g.x)
    assert float(r @ r) / float(_np(bt) @ _np(bt)) <= 1e-10 * (1 + 1e-6)
    # the residual-mode kernel records its iterates too: step for step with the oracle
    g2 = csk.csk_solve(At, bt, nsq, x_star=None, tol=1e-30, max_iters=200, num_ctas=num_ctas,
                       cluster_size=cluster, trace=201, trace_x=True, trace_r=201)
    assert not np.isnan(_np(g2.x_trace)).any()
    _lockstep(At, bt, nsq, g2.x_trace, g2.idx_trace, 200, g2.r_trace)


@pytest.mark.parametrize("m,n,d,kw,resmode", [
    (6000, 40, 400, {}, False),                                   # one 16-CTA cluster (DSMEM exchange)
    (6000, 40, 400, {"num_ctas": 148, "cluster_size": 1}, True),  # grid exchange, residual stop
    (60000, 300, 3000, {}, False),                                # register rows on 148 CTAs
    (40000, 1000, 2000, {"num_ctas": 16, "tmem": True}, False),   # TMEM + shared-memory tiers
])
def test_solve_warm_start(csk, m, n, d, kw, resmode):
    """Algorithm 1 from an arbitrary x0 (INPUT ... x0; the loop P:61-64 is the same from any
    start): the kernel takes x0 from x, and its trajectory follows the oracle's from the same x0 --
    lockstep with r_k, the same i_k sequence and stop."""
    p = make_dense(m, n, "gauss", 900 + n, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, d, seed=11)
    gen = torch.Generator().manual_seed(4242 + n)
    x0 = (torch.randn(n, generator=gen, dtype=torch.float64) * 3.0).to("cuda")
    xs = None if resmode else p.x_star
    cap = 400
    tol = 1e-8 if resmode else 1e-6
    g = csk.csk_solve(At, bt, nsq, x0=x0, x_star=xs, tol=tol, max_iters=cap, trace=cap + 1, trace_x=True,
                      trace_r=80, **kw)
    assert torch.equal(g.x_trace[0], x0), "x_0 is not the given start"
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x0=_np(x0), x_star=None if xs is None else _np(xs),
                     tol=tol, max_iters=cap, trace=cap + 1)
    assert g.termination == o.termination
    assert abs(g.iterations - o.iterations) <= max(1, 0.05 * o.iterations)
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 80, g.r_trace)
    k = min(g.iterations, o.iterations)
    assert np.array_equal(_np(g.idx_trace)[:k], o.idx_trace[:k])


def test_solve_edge_cases(csk):
    dev = "cuda"
    # A = I4, b = (4,3,2,1): exactly 4 steps, indices 0..3
    At = torch.eye(4, dtype=torch.float64, device=dev)
    b = torch.tensor([4.0, 3.0, 2.0, 1.0], dtype=torch.float64, device=dev)
    g = csk.csk_solve(At, b, torch.ones(4, dtype=torch.float64, device=dev), x_star=b,
                      tol=1e-30, trace=10)
    assert g.iterations == 4 and _np(g.idx_trace).tolist() == [0, 1, 2, 3]
    assert torch.equal(g.x, b)
    # x0 = x* -> 0 iterations
    p = make_dense(300, 6, "gauss", 3, dev)
    At, bt, nsq = csk.csk_sketch(p.A, p.b, 40)
    g = csk.csk_solve(At, bt, nsq, x0=p.x_star, x_star=p.x_star)
    assert g.iterations == 0 and g.termination == csk.CONVERGED
    # max_iters = 0 and the cap
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=0)
    assert g.iterations == 0 and g.termination == csk.MAX_ITERS
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=3, tol=1e-30)
    assert g.iterations == 3 and g.termination == csk.MAX_ITERS
    # stagnation: consistent-looking zero residual, RES > tol
    g = csk.csk_solve(torch.tensor([[1.0, 0.0]], dtype=torch.float64, device=dev),
                      torch.zeros(1, dtype=torch.float64, device=dev),
                      torch.ones(1, dtype=torch.float64, device=dev),
                      x_star=torch.tensor([0.0, 1.0], dtype=torch.float64, device=dev))
    assert g.termination == csk.STAGNATED and g.iterations == 0
    # masked zero rows never selected
    At = torch.tensor([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]], dtype=torch.float64, device=dev)
    bt = torch.tensor([100.0, 1.0, 2.0], dtype=torch.float64, device=dev)
    g = csk.csk_solve(At, bt, csk.csk_row_norms(At), x_star=torch.tensor([1.0, 2.0], dtype=torch.float64, device=dev),
                      tol=1e-30, trace=10)
    assert 0 not in _np(g.idx_trace).tolist()
    # zero sketch -> CSK_E_ZERO_SKETCH
    with pytest.raises(csk.CskError) as e:
        z = torch.zeros(3, 2, dtype=torch.float64, device=dev)
        csk.csk_solve(z, torch.ones(3, dtype=torch.float64, device=dev),
                      torch.zeros(3, dtype=torch.float64, device=dev),
                      x_star=torch.ones(2, dtype=torch.float64, device=dev))
    assert e.value.status == csk.CSK_E_ZERO_SKETCH


def test_identity_map_solve_is_mwrk(csk):
    """CSK with d = m, h = id equals MWRK on (A, b) (Remark 1): same i_k sequence."""
    p = make_dense(400, 12, "gauss", 4, "cuda")
    h = torch.arange(400, dtype=torch.int32, device="cuda")
    s = torch.ones(400, dtype=torch.int8, device="cuda")
    s[::3] = -1
    At, bt, nsq = csk.csk_sketch_with_map(p.A, p.b, 400, h, s)
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=1e-12, trace=2000)
    o = oracle.mwrk(_np(p.A), _np(p.b), x_star=_np(p.x_star), tol=1e-12, trace=2000)
    n_same = min(len(g.idx_trace), len(o.idx_trace)) - 2
    assert np.array_equal(_np(g.idx_trace)[:n_same], o.idx_trace[:n_same])


@pytest.mark.parametrize("d,n,num_ctas,smem_rows,tmem,ring", [
    (6000, 150, 8, 0, None, True), (6000, 150, 8, 0, None, False), (5000, 100, 6, -1, None, True),
    (4000, 50, 3, 0, None, True), (3000, 2, 2, 0, None, True), (3000, 64, 1, 0, None, True),
    (2500, 500, 4, 0, None, True), (2500, 500, 4, 3, False, True), (1200, 2000, 6, 0, None, True),
    (900, 2048, 5, 0, None, True), (3001, 130, 5, 0, None, True), (4000, 151, 5, 0, None, True)])
def test_solve_stream_ring(csk, d, n, num_ctas, smem_rows, tmem, ring):
    """Rows past the on-chip tiers through the TMA stream ring (ST variants, loop.cu): stages of
    up to 4 whole rows, several row groups per CTA, ragged last chunks, odd n (plain-load path),
    and the ring disabled (stream_ring=False) -- the same i_k sequence and x_k as the oracle."""
    p = make_dense(d, n, "lognormal_rows", d + n, "cuda")
    At, bt = p.A, p.b
    nsq = csk.csk_row_norms(At)
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, num_ctas=num_ctas, smem_rows=smem_rows, tmem=tmem,
                      stream_ring=ring, trace=200, trace_x=True, trace_r=200, max_iters=200 if n > 1000 else 50000)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star), trace=200,
                     max_iters=200 if n > 1000 else 50000)
    if n <= 1000:
        _free_running(g, o)
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 200, g.r_trace)


@pytest.mark.parametrize("d,n,num_ctas,tmem", [(6000, 150, 8, None), (4000, 50, 3, None), (1200, 2000, 6, None),
                                                (2500, 500, 4, False), (3001, 130, 5, None)])
def test_solve_stream_ring_residual_mode(csk, d, n, num_ctas, tmem):
    """The residual stop (no x*, RES_k = ||b~ - A~ x_k||^2 / ||b~||^2) with streamed rows: the
    RESMODE ring variants give the oracle's i_k and x_k step for step and its stop."""
    p = make_dense(d, n, "lognormal_rows", d + n + 1, "cuda")
    At, bt = p.A, p.b
    nsq = csk.csk_row_norms(At)
    its = 150 if n > 1000 else 50000
    g = csk.csk_solve(At, bt, nsq, x_star=None, tol=1e-12, num_ctas=num_ctas, tmem=tmem, trace=150,
                      trace_x=True, trace_r=150, max_iters=its)
    assert csk.csk_last_solve_tiers()["ring_stages"] >= 2
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=None, tol=1e-12, trace=150, max_iters=its)
    assert g.stop_mode == csk.STOP_RESIDUAL
    if n <= 1000:
        assert g.termination == o.termination == csk.CONVERGED
        assert abs(g.iterations - o.iterations) <= max(1, 0.02 * o.iterations)
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 150, g.r_trace)


@pytest.mark.parametrize("smem_rows,tmem", [(0, None), (-1, False)])
def test_mwrk_unsketched_parity(csk, smem_rows, tmem):
    """MWRK on the unsketched system (Remark 1) = the same loop
    kernel on (A, b, ||A_i||^2) with d = m rows (tmem=False, smem_rows=-1: every row past the
    register tier re-read from L2/HBM each iteration)."""
    p = make_dense(12000, 200, "lognormal_rows", 23, "cuda")
    nsq = csk.csk_row_norms(p.A)
    g = csk.csk_solve(p.A, p.b, nsq, x_star=p.x_star, smem_rows=smem_rows, tmem=tmem, trace=300, trace_x=True,
                      trace_r=100)
    o = oracle.mwrk(_np(p.A), _np(p.b), x_star=_np(p.x_star), trace=300)
    _free_running(g, o)
    _lockstep(p.A, p.b, nsq, g.x_trace, g.idx_trace, 100, g.r_trace)
    _lockstep(p.A, p.b, nsq, g.x_trace, g.idx_trace, 300)


def test_run_and_run_host(csk):
    cfg = CONFIGS["C2"]
    p = make_config(cfg, "cuda")
    x, rep = csk.csk_run(p.A, p.b, cfg.d, x_star=p.x_star)
    assert rep.termination == csk.CONVERGED and rep.final_res <= 1e-6
    xh, reph = csk.csk_run_host(p.A.cpu().pin_memory(), p.b.cpu(), cfg.d, x_star=p.x_star.cpu())
    assert reph.iterations == rep.iterations and torch.equal(xh, x.cpu())


# ---------------------------------------------------------------- full-size configs
def test_C3_full_parity(csk):
    cfg = CONFIGS["C3"]
    p = make_config(cfg, "cuda")
    At, bt, nsq = _check_sketch(csk, p.A, p.b, cfg.d, cfg.sketch_seed)
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cfg.max_iters, trace=2000, trace_x=True,
                      trace_r=2000)
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star),
                     max_iters=cfg.max_iters, trace=2000)
    _free_running(g, o)
    # every iteration of the full C3 solve: r_k within 1e-10, same i_k, x_{k+1} within 1e-12
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, g.iterations, g.r_trace)
    n_same = min(len(g.idx_trace), len(o.idx_trace))
    assert np.array_equal(_np(g.idx_trace)[:n_same], o.idx_trace[:n_same])


def test_residual_sum_complete(csk):
    """Residual stop on one GPU: RES_k = ||r_k||^2/||b~||^2 is summed from the CTA partials beside
    the arrival count and read with one 32-byte load (loop.cu: a hardware property, not a PTX
    guarantee).  Every iteration, the kernel's RES_k must equal the sum over the traced r_k to
    within rounding -- a CTA partial missing from the snapshot would be a ~1/148 deficit."""
    cfg = CONFIGS["C3"]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
    bb = float(_np(bt) @ _np(bt))
    for rep in range(3):
        g = csk.csk_solve(At, bt, nsq, x_star=None, tol=1e-30, max_iters=600, trace=601, trace_r=601)
        r = _np(g.r_trace)
        want = np.einsum("ij,ij->i", r, r) / bb
        got = _np(g.res_trace)
        assert len(got) == len(want) == 601
        assert np.all(np.abs(got - want) <= 1e-12 * want), (rep, np.max(np.abs(got - want) / want))


def test_C4_full_size_sampled(csk):
    """8 GB A: sampled buckets against the oracle's fold of exactly those rows; the first 3 000
    iterations free-running on both sides (the oracle on the GPU's A~, ~45 s): the same i_k
    sequence, both MaxIters, RES within 1e-6 relative (SURVEY §8(c) acceptance 4 at a 3 000 cap);
    lockstep with the r_k trace on the first iterations; and properties over the whole
    50k-iteration run (monotone RES, eq:A).  The full 50k comparison against the oracle is the
    committed artifact profiles/r02_parity_C4.txt (tools/parity_full.py)."""
    cfg = CONFIGS["C4"]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
    torch.cuda.synchronize()
    h, s = oracle.hash_map(cfg.sketch_seed, cfg.m, cfg.d)
    rng = np.random.default_rng(0)
    for j in rng.choice(cfg.d, 24, replace=False).tolist() + [0, cfg.d - 1]:
        rows = np.nonzero(h == j)[0]
        sub = _np(p.A[torch.as_tensor(rows, device="cuda")]) if len(rows) else np.zeros((0, cfg.n))
        bsub = _np(p.b[torch.as_tensor(rows, device="cuda")]) if len(rows) else np.zeros(0)
        if len(rows):
            a1, b1 = oracle.sketch_dense(sub, bsub, 1, h=np.zeros(len(rows), np.int32), s=s[rows])
        else:
            a1, b1 = np.zeros((1, cfg.n)), np.zeros(1)
        assert np.array_equal(_np(At[j]), a1[0]) and _np(bt[j]) == b1[0]
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cfg.max_iters, trace=cfg.max_iters + 1)
    assert g.termination in (csk.CONVERGED, csk.MAX_ITERS)
    res = _np(g.res_trace)
    assert np.all(np.diff(res) <= 1e-12 * res[:-1])
    g20 = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=12, tol=1e-30, trace=13, trace_x=True, trace_r=13)
    _lockstep(At, bt, nsq, g20.x_trace, g20.idx_trace, 12, g20.r_trace)
    assert np.array_equal(_np(g20.idx_trace), _np(g.idx_trace)[:12])
    # free-running at a 3 000-iteration cap on both sides
    cap = 3000
    g3 = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, trace=cap + 1)
    Atn, btn = _np(At), _np(bt)
    o3 = oracle.solve(Atn, btn, oracle.row_norms(Atn), x_star=_np(p.x_star), max_iters=cap, trace=cap + 1)
    assert g3.termination == o3.termination == csk.MAX_ITERS and g3.iterations == o3.iterations == cap
    assert np.array_equal(_np(g3.idx_trace), o3.idx_trace)
    assert abs(g3.final_res - o3.final_res) <= 1e-6 * o3.final_res
    assert np.allclose(_np(g3.res_trace), o3.res_trace, rtol=1e-6, atol=0)


# ---------------------------------------------------------------- CSR input (config C5)
def _csr_np(p):
    return _np(p.row_ptr), _np(p.col), _np(p.val), _np(p.b)


@pytest.mark.parametrize("m,n,d,k", [(3000, 64, 300, 5), (20000, 2000, 1000, 10), (4001, 33, 777, 7)])
def test_sketch_csr_bitexact(csk, m, n, d, k):
    from csk_synth import make_csr
    p = make_csr(m, n, k, seed=31 + m, device="cuda")
    At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, n, d, seed=5)
    rp, col, val, b = _csr_np(p)
    At_o, bt_o = oracle.sketch_csr(rp, col, val, b, n, d, seed=5)
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
    assert np.array_equal(_np(nsq), oracle.row_norms(At_o))


@pytest.mark.parametrize("m,n,d,maxlen", [(5000, 300, 400, 70), (3000, 1500, 50, 40), (2000, 1500, 30, 700),
                                           (4000, 2001, 3999, 1200), (600, 64, 7, 64)])
def test_sketch_csr_ragged_rows(csk, m, n, d, maxlen):
    """CSR rows of 0..maxlen stored pairs (empty rows and buckets, rows longer than one 256-pair
    gather stage -- split over several batches --, many rows per bucket, odd n, unsorted bucket
    sizes): the staged CSR kernel folds every column in ascending row order."""
    g = np.random.default_rng(m + n)
    lens = g.integers(0, maxlen + 1, size=m)
    lens[::97] = 0
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(g.choice(n, size=int(k), replace=False)) for k in lens]).astype(np.int32)
    val = g.standard_normal(int(rp[-1]))
    b = g.standard_normal(m)
    At, bt, nsq = csk.csk_sketch_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(),
                                     torch.from_numpy(val).cuda(), torch.from_numpy(b).cuda(), n, d, seed=13)
    At_o, bt_o = oracle.sketch_csr(rp, col, val, b, n, d, seed=13)
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
    assert np.array_equal(_np(nsq), oracle.row_norms(At_o))


def test_C5_full_size_sampled(csk):
    """4e6 x 2000 CSR (4e7 nnz): sampled buckets against the oracle's fold of exactly those
    rows; the first iterations in lockstep against the oracle's residual."""
    cfg = CONFIGS["C5"]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, cfg.n, cfg.d, seed=cfg.sketch_seed)
    torch.cuda.synchronize()
    h, s = oracle.hash_map(cfg.sketch_seed, cfg.m, cfg.d)
    rp = _np(p.row_ptr)
    rng = np.random.default_rng(1)
    for j in rng.choice(cfg.d, 16, replace=False).tolist() + [0, cfg.d - 1]:
        rows = np.nonzero(h == j)[0]
        if not len(rows):
            assert not _np(At[j]).any() and _np(bt[j]) == 0.0
            continue
        sub_rp = np.concatenate([[0], np.cumsum(rp[rows + 1] - rp[rows])]).astype(np.int64)
        idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
        cols = _np(p.col[torch.as_tensor(idx, device="cuda")])
        vals = _np(p.val[torch.as_tensor(idx, device="cuda")])
        bs = _np(p.b[torch.as_tensor(rows, device="cuda")])
        a1, b1 = oracle.sketch_csr(sub_rp, cols, vals, bs, cfg.n, 1, h=np.zeros(len(rows), np.int32), s=s[rows])
        assert np.array_equal(_np(At[j]), a1[0]) and _np(bt[j]) == b1[0]
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=6, tol=1e-30, trace=7, trace_x=True, trace_r=7)
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 6, g.r_trace)
    # the residual stop at full size (x* unknown): streamed rows through the RESMODE ring
    g = csk.csk_solve(At, bt, nsq, x_star=None, max_iters=6, tol=1e-30, trace=7, trace_x=True, trace_r=7)
    assert g.stop_mode == csk.STOP_RESIDUAL and csk.csk_last_solve_tiers()["ring_stages"] >= 2
    _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, 6, g.r_trace)

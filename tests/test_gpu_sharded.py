"""GPU tests of the sharded path (S9/S10) on one B200.

* csk_solve_virtual_ranks runs the production candidate/apply kernels for P virtual ranks with
  a loopback exchange: every virtual rank must end with bit-identical x, and the trajectory
  must match the oracle (lockstep bar: same i_k, iteration count within 5 %).
* csk_comm_create with a 1-rank NCCL communicator drives csk_sketch_sharded (ncclReduceScatter)
  and csk_solve_sharded (ncclAllGather) through real NCCL on one GPU; with P = 1 the
  reduce-scatter is an identity, so A~ must be bit-exact with the oracle.
Real P > 1 NCCL runs need P GPUs (bench.py under torchrun).
"""
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import oracle
from csk_synth import CONFIGS, make_config, make_dense

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def csk():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2004_02480_b200 as m
    return m


def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_virtual_ranks_match_oracle(csk, P):
    """The S10 decomposition (P virtual ranks, one launch) against the oracle step for step: the
    same i_k sequence, every rank's r_k (traced by global row) within 1e-10 of the oracle's
    r(x_k), x_{k+1} within 1e-12 (the lockstep bar of test_gpu_parity.py)."""
    from test_gpu_parity import _lockstep
    cfg = CONFIGS["C2"]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
    x, copies, rep, tr = csk.csk_solve_virtual_ranks(At, bt, nsq, P, x_star=p.x_star, tol=cfg.tol,
                                                     max_iters=cfg.max_iters, trace=2000, trace_x=True,
                                                     trace_r=2000)
    assert all(torch.equal(copies[q], copies[0]) for q in range(P))
    assert torch.equal(x, copies[0])
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(p.x_star), tol=cfg.tol,
                     max_iters=cfg.max_iters, trace=2000)
    assert rep.termination == csk.CONVERGED and rep.final_res <= cfg.tol
    assert abs(rep.iterations - o.iterations) <= max(1, 0.05 * o.iterations)
    n_same = min(len(tr.idx_trace), len(o.idx_trace))
    assert np.array_equal(_np(tr.idx_trace)[:n_same], o.idx_trace[:n_same])
    assert not np.isnan(_np(tr.r_trace)).any()  # every rank wrote its rows
    _lockstep(At, bt, nsq, tr.x_trace, tr.idx_trace, rep.iterations, tr.r_trace)
    # the single-GPU persistent kernel and the sharded kernels agree on the trajectory length
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=cfg.tol, max_iters=cfg.max_iters)
    assert abs(g.iterations - rep.iterations) <= max(1, 0.05 * o.iterations)


def test_virtual_ranks_c4_layout(csk):
    """The SYS kernel with C4's per-CTA layout (4-warp groups of 6 register + 16 TMEM + 12
    shared-memory rows: the fused TMEM + shared-memory pass) in a 2-rank decomposition: the
    oracle's i_k sequence, r_k within the lockstep bar, identical copies of x."""
    from test_gpu_parity import _lockstep
    P, n = 2, 1000
    d = P * 74 * 68  # 74 CTAs per virtual rank, 68 rows each
    g = torch.Generator(device="cuda").manual_seed(2468)
    At = torch.randn(d, n, dtype=torch.float64, device="cuda", generator=g)
    xs = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    bt = At @ xs
    nsq = csk.csk_row_norms(At)
    cap = 80
    x, copies, rep, tr = csk.csk_solve_virtual_ranks(At, bt, nsq, P, x_star=xs, tol=1e-30, max_iters=cap,
                                                     trace=cap + 1, trace_x=True, trace_r=20)
    t = csk.csk_last_solve_tiers()
    assert (t["group_warps"], t["reg_rows"], t["tmem_rows"], t["smem_rows"]) == (4, 6, 16, 12), t
    assert all(torch.equal(copies[q], copies[0]) for q in range(P))
    o = oracle.solve(_np(At), _np(bt), oracle.row_norms(_np(At)), x_star=_np(xs), tol=1e-30, max_iters=cap,
                     trace=cap + 1)
    assert rep.termination == o.termination == csk.MAX_ITERS
    assert np.array_equal(_np(tr.idx_trace)[:cap], o.idx_trace[:cap])
    _lockstep(At, bt, nsq, tr.x_trace, tr.idx_trace, 20, tr.r_trace)


@pytest.mark.parametrize("P", [2, 4])
def test_virtual_ranks_streamed_rows(csk, P):
    """Rows past the on-chip tiers (92 MB of A > what 148 SMs hold) stream through the TMA ring
    inside the P-rank decomposition too (MWRK on a tall system, Remark 1)."""
    p = make_dense(90000, 128, "lognormal_rows", 31, "cuda")
    nsq = csk.csk_row_norms(p.A)
    x, copies, rep, tr = csk.csk_solve_virtual_ranks(p.A, p.b, nsq, P, x_star=p.x_star, tol=1e-6, max_iters=5000,
                                                     trace=5001)
    assert all(torch.equal(copies[q], copies[0]) for q in range(P))
    o = oracle.mwrk(_np(p.A), _np(p.b), x_star=_np(p.x_star), tol=1e-6, max_iters=5000, trace=5001)
    assert rep.termination == csk.CONVERGED and rep.final_res <= 1e-6
    assert abs(rep.iterations - o.iterations) <= max(1, 0.05 * o.iterations)
    n_same = min(len(tr.idx_trace), len(o.idx_trace))
    assert np.array_equal(_np(tr.idx_trace)[:n_same], o.idx_trace[:n_same])
    # the residual stop (x* unknown) through the ring's SYS twins: the partials cross ranks
    x, copies, rep = csk.csk_solve_virtual_ranks(p.A, p.b, nsq, P, x_star=None, tol=1e-12, max_iters=5000)
    assert all(torch.equal(copies[q], copies[0]) for q in range(P))
    o = oracle.mwrk(_np(p.A), _np(p.b), x_star=None, tol=1e-12, max_iters=5000)
    assert rep.stop_mode == csk.STOP_RESIDUAL and rep.termination == o.termination == csk.CONVERGED
    assert abs(rep.iterations - o.iterations) <= max(1, 0.05 * o.iterations)


def test_virtual_ranks_residual_mode_and_cap(csk):
    p = make_dense(6000, 40, "gauss", 12, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, 400, seed=2)
    x, _, rep = csk.csk_solve_virtual_ranks(At, bt, nsq, 3, x_star=None, tol=1e-10)
    assert rep.stop_mode == csk.STOP_RESIDUAL and rep.termination == csk.CONVERGED
    r = _np(bt) - _np(At) @ _np(x)
    assert float(r @ r) / float(_np(bt) @ _np(bt)) <= 1e-10 * (1 + 1e-6)
    _, _, rep = csk.csk_solve_virtual_ranks(At, bt, nsq, 4, x_star=p.x_star, tol=1e-30, max_iters=5)
    assert rep.termination == csk.MAX_ITERS and rep.iterations == 5


def test_one_rank_nccl_sketch_and_solve(csk):
    cfg = CONFIGS["C2"]
    p = make_config(cfg, "cuda")
    ctx = csk.Context()
    csk.comm_create(csk.comm_unique_id(), 1, 0, ctx=ctx)
    At, bt, nsq, lo, hi = csk.csk_sketch_sharded(p.A, p.b, 0, cfg.m, cfg.d, 1, 0, seed=cfg.sketch_seed, ctx=ctx)
    assert (lo, hi) == (0, cfg.d)
    At_o, bt_o = oracle.sketch_dense(_np(p.A), _np(p.b), cfg.d, seed=cfg.sketch_seed)
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
    x, rep = csk.csk_solve_sharded(At, bt, nsq, lo, hi, cfg.d, cfg.n, x_star=p.x_star, tol=cfg.tol,
                                   max_iters=cfg.max_iters, ctx=ctx)
    o = oracle.solve(At_o, bt_o, oracle.row_norms(At_o), x_star=_np(p.x_star), tol=cfg.tol,
                     max_iters=cfg.max_iters)
    assert rep.termination == csk.CONVERGED
    assert abs(rep.iterations - o.iterations) <= max(1, 0.05 * o.iterations)
    csk.comm_destroy(ctx)


def test_one_rank_nccl_row_offset_shard(csk):
    """A rank holding rows [lo, hi) of A with row_offset = lo hashes them with global indices:
    its partial equals the oracle fold of exactly those rows under the global map."""
    m, n, d = 5000, 30, 300
    p = make_dense(m, n, "gauss", 4, "cuda")
    ctx = csk.Context()
    csk.comm_create(csk.comm_unique_id(), 1, 0, ctx=ctx)
    lo, hi = 1234, 4321
    At, bt, _, _, _ = csk.csk_sketch_sharded(p.A[lo:hi].contiguous(), p.b[lo:hi].contiguous(), lo, m, d, 1, 0,
                                             seed=9, ctx=ctx)
    h, s = oracle.hash_map(9, m, d)
    At_o, bt_o = oracle.sketch_dense(_np(p.A)[lo:hi], _np(p.b)[lo:hi], d, h=h[lo:hi], s=s[lo:hi])
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
    csk.comm_destroy(ctx)


def test_bench_sharded_path_one_rank(csk):
    """bench.py's N > 1 path (S9 + S10 through NCCL, the fused peer-memory loop, its roofline
    and e2e keys) run through a 1-rank communicator on this GPU."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_PORT="29631")
    out = subprocess.run([sys.executable, "bench.py", "--sharded", "--steps", "2", "--warmup", "3", "--no-extras",
                          "--no-cpu"], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["termination"] == "converged" and d["final_res"] <= 1e-6
    for key in ("metric", "value", "unit", "n_gpus", "ms_per_step", "scaling", "config", "clocks", "e2e", "roofline",
                "gpu_launches"):
        assert key in d, key
    assert d["roofline"]["kernel_ms"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0


# ---------------------------------------------------------------- S9 for CSR (config C5)
def _csr(m, n, d, k, seed, ragged=False):
    from csk_synth import make_csr
    if not ragged:
        p = make_csr(m, n, k, seed=seed, device="cuda")
        return p.row_ptr, p.col, p.val, p.b
    g = np.random.default_rng(seed)
    lens = g.integers(0, k + 1, size=m)
    lens[::53] = 0
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(g.choice(n, size=int(x), replace=False)) for x in lens]).astype(np.int32)
    val = g.standard_normal(int(rp[-1]))
    b = g.standard_normal(m)
    return (torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(),
            torch.from_numpy(b).cuda())


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("m,n,d,k,ragged", [(20000, 300, 1000, 10, False), (5000, 200, 61, 40, True),
                                           (3000, 64, 8, 12, True)])
def test_csr_row_routing_virtual_bitexact(csk, P, m, n, d, k, ragged):
    """S9 by row routing: P contiguous row shards, every row sent to its bucket's
    owner, owners fold in ascending global row order -> A~, b~ identical to the single-GPU sketch and
    to the oracle (P virtual ranks on this GPU: the packing, segment order and owner-side plan are
    the production kernels; only the transport is a device copy instead of NCCL)."""
    rp, col, val, b = _csr(m, n, d, k, 100 + m + P, ragged)
    At, bt, nsq = csk.csk_sketch_csr_routed_virtual(rp, col, val, b, n, d, P, seed=7)
    At1, bt1, nsq1 = csk.csk_sketch_csr(rp, col, val, b, n, d, seed=7)
    assert torch.equal(At, At1) and torch.equal(bt, bt1) and torch.equal(nsq, nsq1)
    At_o, bt_o = oracle.sketch_csr(_np(rp), _np(col), _np(val), _np(b), n, d, seed=7)
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)


@pytest.mark.parametrize("mode", [0, 1])
def test_one_rank_nccl_csr_sharded(csk, mode):
    """csk_sketch_csr_sharded through a real 1-rank NCCL communicator, both modes (reduce-scatter
    of partial A~; row routing with ncclSend/ncclRecv to self): bit-exact with the oracle at P = 1,
    for a shard that is a row slice of a larger matrix (global hashing via row_offset)."""
    m, n, d = 12000, 250, 700
    rp, col, val, b = _csr(m, n, d, 10, 5)
    ctx = csk.Context()
    csk.comm_create(csk.comm_unique_id(), 1, 0, ctx=ctx)
    lo, hi = 2500, 9100  # this "rank" holds rows [lo, hi) of the global matrix
    At, bt, nsq, dlo, dhi = csk.csk_sketch_csr_sharded(rp[lo:hi + 1], col, val, b[lo:hi], lo, m, n, d, 1, 0,
                                                       seed=3, mode=mode, ctx=ctx)
    assert (dlo, dhi) == (0, d)
    h, s = oracle.hash_map(3, m, d)
    sub_rp = (_np(rp)[lo:hi + 1] - _np(rp)[lo]).astype(np.int64)
    a0 = int(_np(rp)[lo])
    At_o, bt_o = oracle.sketch_csr(sub_rp, _np(col)[a0:], _np(val)[a0:], _np(b)[lo:hi], n, d, h=h[lo:hi], s=s[lo:hi])
    assert np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
    csk.comm_destroy(ctx)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (real NCCL peers)")
def test_two_gpu_nccl_parity():
    """>= 2 GPUs: torchrun the sharded bench path at N = 2 (S9 dense + CSR routing, S10 over peer
    memory) and check its solves reach the oracle-equivalent stop (the bench asserts parity flags)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-extras",
                          "--no-cpu", "--no-e2e"], cwd=root, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    dd = json.loads(out.stdout.strip().splitlines()[-1])
    assert dd["n_gpus"] == 2 and dd["termination"] == "converged"

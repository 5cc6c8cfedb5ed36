"""Multi-process (gloo, world_size 2, CPU) tests of the sharded path's host logic (S9/S10).

What runs on the GPU -- the sketch / candidate / apply kernels and the NCCL collectives --
cannot run here.  These tests check, on two real processes, everything around them:
  * the NCCL unique-id bootstrap over torch.distributed (paper_2004_02480_b200.parallel);
  * bucket ownership (csk_shard_range) and input-row shards cover [0, d) / [0, m) exactly once;
  * the sharded decomposition itself, evaluated with the CPU oracle as the local step:
    partial sketches of row shards hashed with GLOBAL row indices sum to the unsharded sketch
    (the ncclReduceScatter of S9), and the per-iteration exchange rule -- every rank's local
    (score, global row, lambda, row) candidate, gathered and resolved by (score desc, row asc)
    -- reproduces the unsharded oracle trajectory step for step (the ncclAllGather of S10).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from csk_synth import make_dense

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(fn, port, world=WORLD):
    mp.spawn(_entry, args=(fn, port, world), nprocs=world, join=True)


def _entry(rank, fn, port, world):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
    finally:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- workers
def _w_uid(rank, world):
    import paper_2004_02480_b200 as csk
    from paper_2004_02480_b200.parallel import broadcast_uid
    uid = csk.comm_unique_id() if rank == 0 else None
    got = broadcast_uid(uid, None, "cpu")
    assert len(got) == 128
    allg = [None] * world
    dist.all_gather_object(allg, got)
    assert all(g == allg[0] for g in allg)
    if rank == 0:
        assert got == uid


def _w_ranges(rank, world):
    import paper_2004_02480_b200 as csk
    from paper_2004_02480_b200.parallel import row_shard
    for d in [1, 7, 500, 5000, 40001]:
        lo, hi = csk.shard_range(d, world, rank)
        got = [None] * world
        dist.all_gather_object(got, (lo, hi))
        cover = np.zeros(d, int)
        for a, b in got:
            cover[a:b] += 1
        assert np.all(cover == 1)
        chunk = (d + world - 1) // world
        assert all(b - a <= chunk for a, b in got)
    for m in [3, 1000, 100001]:
        got = [None] * world
        dist.all_gather_object(got, row_shard(m, world, rank))
        assert got[0][0] == 0 and got[-1][1] == m and all(got[i][1] == got[i + 1][0] for i in range(world - 1))


def _w_sketch_decomposition(rank, world):
    from paper_2004_02480_b200.parallel import row_shard
    m, n, d, seed = 3000, 24, 301, 17
    p = make_dense(m, n, "lognormal_rows", 5, "cpu")
    A, b = p.A.numpy(), p.b.numpy()
    h, s = oracle.hash_map(seed, m, d)           # global map: rank shards slice it
    lo, hi = row_shard(m, world, rank)
    At_p, bt_p = oracle.sketch_dense(A[lo:hi], b[lo:hi], d, h=h[lo:hi], s=s[lo:hi])
    t = torch.from_numpy(np.concatenate([At_p.reshape(-1), bt_p]))
    dist.all_reduce(t)                            # stands in for ncclReduceScatter(sum)
    At_full, bt_full = oracle.sketch_dense(A, b, d, seed=seed)
    At_sum = t[: d * n].numpy().reshape(d, n)
    bt_sum = t[d * n:].numpy()
    # both are recursive sums of the same c_j terms in different association: each within
    # (c_j + world - 1) u sum|a| of the exact sum, so they differ by <= 2 (c_j + world) u sum|a|
    c = np.bincount(h, minlength=d).astype(float)
    absA = np.zeros((d, n))
    np.add.at(absA, h, np.abs(A))
    u = 2.0**-53
    assert np.all(np.abs(At_sum - At_full) <= 2 * (c[:, None] + world) * u * absA + 1e-300)
    absb = np.zeros(d)
    np.add.at(absb, h, np.abs(b))
    assert np.all(np.abs(bt_sum - bt_full) <= 2 * (c + world) * u * absb + 1e-300)
    assert np.array_equal(At_sum == 0, absA == 0)
    # owner slice as csk_shard_range assigns it
    import paper_2004_02480_b200 as csk
    dlo, dhi = csk.shard_range(d, world, rank)
    assert At_sum[dlo:dhi].shape == (dhi - dlo, n)


def _w_loop_decomposition(rank, world):
    import paper_2004_02480_b200 as csk
    m, n, d = 4000, 30, 400
    p = make_dense(m, n, "gauss", 8, "cpu")
    At, bt = oracle.sketch_dense(p.A.numpy(), p.b.numpy(), d, seed=3)
    nsq = oracle.row_norms(At)
    xs = p.x_star.numpy()
    ref = oracle.solve(At, bt, nsq, x_star=xs, tol=1e-10, trace=5000)
    lo, hi = csk.shard_range(d, world, rank)
    x = np.zeros(n)
    it = 0
    while True:
        e = x - xs
        res = float(e @ e) / float(xs @ xs)
        if res <= 1e-10:
            break
        r = oracle.residual(At[lo:hi], bt[lo:hi], x)
        sc = np.where(nsq[lo:hi] > 0, r * r / np.where(nsq[lo:hi] > 0, nsq[lo:hi], 1), -1.0)
        li = int(np.argmax(sc))
        rec = torch.tensor([sc[li], lo + li, r[li] / nsq[lo + li]] + list(At[lo + li]), dtype=torch.float64)
        got = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(got, rec)                 # stands in for ncclAllGather (S10)
        best = None
        for g in got:                             # rank order; (score desc, global row asc)
            key = (-float(g[0]), int(g[1]))
            if best is None or key < best[0]:
                best = (key, g)
        g = best[1]
        assert int(g[1]) == int(ref.idx_trace[it]), (it, int(g[1]), int(ref.idx_trace[it]))
        x = x + float(g[2]) * g[3:].numpy()
        it += 1
    assert abs(it - ref.iterations) <= 1


def _w_csr_routing(rank, world):
    """S9 for CSR by row routing (csk_sketch_csr_sharded, CSK_SHARD_ROUTE_ROWS): every input row goes
    to the owner of its bucket (owner = h // ceil(d/P), csk_shard_range), rows leave each rank in
    ascending order and are concatenated in source-rank order; each owner's fold of what it received
    equals the single-process sketch of its bucket rows BIT FOR BIT (ragged CSR, empty rows)."""
    import paper_2004_02480_b200 as csk
    from paper_2004_02480_b200.parallel import row_shard
    m, n, d, seed = 2500, 40, 97, 21
    g = np.random.default_rng(77)
    lens = g.integers(0, 12, size=m)
    lens[::41] = 0
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(g.choice(n, size=int(x), replace=False)) for x in lens]).astype(np.int32)
    val = g.standard_normal(int(rp[-1]))
    b = g.standard_normal(m)
    h, sg = oracle.hash_map(seed, m, d)
    chunk = -(-d // world)
    lo, hi = row_shard(m, world, rank)
    send = [[(i, b[i], col[rp[i]:rp[i + 1]].tolist(), val[rp[i]:rp[i + 1]].tolist())
             for i in range(lo, hi) if h[i] // chunk == q] for q in range(world)]
    allsend = [None] * world
    dist.all_gather_object(allsend, send)          # stands in for the grouped ncclSend/ncclRecv
    recv = [r for src in range(world) for r in allsend[src][rank]]
    rows = np.array([r[0] for r in recv], np.int64)
    assert np.all(np.diff(rows) > 0)               # ascending global rows at the owner
    dlo, dhi = csk.shard_range(d, world, rank)
    sub_rp = np.zeros(len(recv) + 1, np.int64)
    sub_rp[1:] = np.cumsum([len(r[2]) for r in recv])
    scol = np.array([c for r in recv for c in r[2]], np.int32)
    sval = np.array([v for r in recv for v in r[3]], np.float64)
    sb = np.array([r[1] for r in recv], np.float64)
    At_o, bt_o = oracle.sketch_csr(sub_rp, scol, sval, sb, n, dhi - dlo,
                                   h=(h[rows] - dlo).astype(np.int32), s=sg[rows])
    At_full, bt_full = oracle.sketch_csr(rp, col, val, b, n, d, seed=seed)
    assert np.array_equal(At_o, At_full[dlo:dhi]) and np.array_equal(bt_o, bt_full[dlo:dhi])


@pytest.mark.parametrize("fn", [_w_uid, _w_ranges, _w_sketch_decomposition, _w_loop_decomposition, _w_csr_routing],
                         ids=["uid_bootstrap", "ownership", "sketch_reduce_scatter", "loop_allgather",
                              "csr_row_routing"])
def test_two_rank_gloo(fn):
    _run(fn, _free_port())

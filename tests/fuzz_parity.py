"""Randomised parity sweep against the oracle (seeded; not part of the default test run).

python tests/fuzz_parity.py [count] [seed]

For each random case: m, n, d, the input kind, and the solve's launch options (grid, cluster,
resident rows, TMEM tier, stream ring) are drawn; the sketch must be bit-exact against the oracle
and the solve must follow the oracle step for step (the lockstep bar of tests/test_gpu_parity.py)
for its first iterations, and reach the same stop as a free-running oracle when that is cheap.
Prints one line per case and a summary; exits 1 on the first failure.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import make_dense  # noqa: E402
from test_gpu_parity import _lockstep, _np  # noqa: E402


def case(rng, k):
    n = int(rng.choice([1, 2, 3, 17, 50, 64, 100, 127, 150, 200, 256, 257, 333, 500, 512, 777, 1000, 1500, 2048]))
    m = int(rng.integers(max(n + 2, 64), max(n + 3, min(200000, 20_000_000 // max(n, 1)))))
    d = int(rng.integers(max(1, n // 2), m))
    d = max(1, min(d, m - 1, 60000))
    kind = str(rng.choice(["gauss", "lognormal_rows", "illcond"]))
    opts = {}
    r = rng.random()
    if r < 0.2:
        opts["num_ctas"] = int(rng.integers(1, 149))
    if rng.random() < 0.2:
        opts["cluster_size"] = int(rng.choice([1, 16]))
    if rng.random() < 0.2:
        opts["smem_rows"] = int(rng.choice([-1, 0, 3, 17]))
    if rng.random() < 0.2:
        opts["tmem"] = bool(rng.random() < 0.5)
    if rng.random() < 0.15:
        opts["stream_ring"] = False
    return m, n, d, kind, opts


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 12345
    rng = np.random.default_rng(seed)
    t0 = time.time()
    for k in range(count):
        m, n, d, kind, opts = case(rng, k)
        p = make_dense(m, n, kind, 7000 + k, "cuda")
        At, bt, nsq = csk.csk_sketch(p.A, p.b, d, seed=k)
        At_o, bt_o = oracle.sketch_dense(_np(p.A), _np(p.b), d, seed=k)
        ok_sk = np.array_equal(_np(At), At_o) and np.array_equal(_np(bt), bt_o)
        if not ok_sk:
            print(f"FAIL sketch case {k}: m={m} n={n} d={d} kind={kind}", flush=True)
            sys.exit(1)
        # a random CSR input of the same shape (0..maxlen stored pairs per row), bit-exact too
        if rng.random() < 0.3 and n >= 2:
            maxlen = int(min(n, rng.integers(1, 80)))
            mm = int(min(m, 30000))
            lens = rng.integers(0, maxlen + 1, size=mm)
            rp = np.zeros(mm + 1, np.int64)
            rp[1:] = np.cumsum(lens)
            col = np.concatenate([np.sort(rng.choice(n, size=int(c), replace=False)) for c in lens]).astype(np.int32) \
                if rp[-1] else np.zeros(0, np.int32)
            val = rng.standard_normal(int(rp[-1]))
            bb = rng.standard_normal(mm)
            dd = int(max(1, min(d, mm - 1)))
            Atc, btc, _ = csk.csk_sketch_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(),
                                             torch.from_numpy(val).cuda(), torch.from_numpy(bb).cuda(), n, dd, seed=k)
            Ao, bo = oracle.sketch_csr(rp, col, val, bb, n, dd, seed=k)
            if not (np.array_equal(_np(Atc), Ao) and np.array_equal(_np(btc), bo)):
                print(f"FAIL csr case {k}: m={mm} n={n} d={dd} maxlen={maxlen}", flush=True)
                sys.exit(1)
            del Atc, btc
        iters = 40
        xs = p.x_star if rng.random() < 0.85 else None  # residual mode sometimes
        try:
            g = csk.csk_solve(At, bt, nsq, x_star=xs, tol=1e-30, max_iters=iters, trace=iters + 1,
                              trace_x=True, **opts)
        except csk.CskError as e:
            if e.status == csk.CSK_E_UNSUPPORTED:
                print(f"case {k}: m={m} n={n} d={d} {opts}: unsupported ({e})", flush=True)
                continue
            if e.status == csk.CSK_E_ZERO_SKETCH:
                continue
            raise
        _lockstep(At, bt, nsq, g.x_trace, g.idx_trace, iters)
        geo = csk.csk_last_solve_tiers()
        print(f"case {k}: m={m} n={n} d={d} kind={kind} opts={opts} ok "
              f"(G={geo['num_ctas']} cl={geo['cluster_size']} rr={geo['reg_rows']} rt={geo['tmem_rows']} "
              f"rs={geo['smem_rows']} ring={geo['ring_stages']}x{geo['ring_rows']})", flush=True)
        del p, At, bt, nsq
        torch.cuda.empty_cache()
    print(f"all {count} cases passed in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()

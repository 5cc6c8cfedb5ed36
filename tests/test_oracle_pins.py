"""Pins for the CPU oracle (oracle/), checked against what the paper and mathematics fix.

None of these compares the oracle with itself: each pin is a published vector, a
value printed in the paper, Definition 1 multiplied out by brute force, a SPEC
worked example, a closed form, or an identity/inequality from the paper's proof
(eq:A, eq:5, eq:6, Theorem 2) evaluated independently in numpy.
Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from csk_synth import make_dense

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MASK64 = 2**64 - 1
GAMMA = 0x9E3779B97F4A7C15


def _golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def _rng_problem(m, n, seed, kind="gauss"):
    p = make_dense(m, n, kind, seed, "cpu")
    return p.A.numpy(), p.b.numpy(), p.x_star.numpy()


# ---------------------------------------------------------------- O-1 PRNG / hash
def test_splitmix64_published_vector():
    want = [int(t[0], 16) for t in _golden_lines("splitmix64_seed0.txt")]
    assert oracle.splitmix64_stream(0, 4) == want


def test_hash_survey_vectors_seed0_d500():
    rows = {t[0]: t[1:] for t in _golden_lines("hash_seed0_d500.txt")}
    h, s = oracle.hash_map(0, 1000, 500)
    assert h[:12].tolist() == [int(v) for v in rows["h"]]
    assert s[:12].tolist() == [1 if v == "+" else -1 for v in rows["s"]]
    cnt = np.bincount(h, minlength=500)
    assert int((cnt == 0).sum()) == int(rows["c1_empty"][0])
    assert int(cnt.max()) == int(rows["c1_max_bucket"][0])
    assert int(s.sum()) == int(rows["c1_sign_sum"][0])
    h2, _ = oracle.hash_map(0, 20000, 2000)
    c2 = np.bincount(h2, minlength=2000)
    assert int((c2 == 0).sum()) == int(rows["c2_empty"][0])
    assert int(c2.max()) == int(rows["c2_max_bucket"][0])


def test_hash_golden_file_matches_its_generator():
    """The golden file's data lines are exactly what the committed big-int script prints."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_hash", os.path.join(GOLDEN, "gen_hash_seed0_d500.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    with open(os.path.join(GOLDEN, "hash_seed0_d500.txt")) as f:
        data = [ln.rstrip("\n") for ln in f if ln.strip() and not ln.startswith("#")]
    assert data == gen.golden_lines()


def _mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


@pytest.mark.parametrize("seed,d", [(0, 500), (12345, 7), (2**63 + 11, 40000), (MASK64, 1)])
def test_hash_counter_form_equals_sequential(seed, d):
    """Counter form SM64(seed, c) = mix(seed + (c+1)*gamma), c = 2i (h) / 2i+1 (sign)."""
    m = 257
    h, s = oracle.hash_map(seed, m, d)
    for i in range(m):
        zh = _mix((seed + (2 * i + 1) * GAMMA) & MASK64)
        zs = _mix((seed + (2 * i + 2) * GAMMA) & MASK64)
        assert h[i] == (zh * d) >> 64
        assert s[i] == (-1 if zs >> 63 else 1)


def test_hash_distribution_def1():
    """h(i) uniform on [d], D_ii = +-1 with probability 1/2."""
    m, d = 400_000, 64
    h, s = oracle.hash_map(7, m, d)
    assert h.min() >= 0 and h.max() < d
    assert set(np.unique(s).tolist()) == {-1, 1}
    cnt = np.bincount(h, minlength=d)
    chi2 = float(((cnt - m / d) ** 2 / (m / d)).sum())
    assert chi2 < 120.0          # 63 dof: P(chi2 > 120) < 1e-5
    assert abs(float(s.sum())) < 5 * np.sqrt(m)


# ---------------------------------------------------------------- O-2 sketch
def test_sketch_equals_dense_definition_bitwise():
    """A~ = (Phi D) A from the explicit d x m matrix of Def. 1, row-order sums."""
    rng = np.random.default_rng(3)
    for trial in range(200):
        m = int(rng.integers(2, 50))
        d = int(rng.integers(1, min(m, 20) + 1))
        n = int(rng.integers(1, 11))
        A = rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, 1)))
        b = rng.standard_normal(m)
        seed = int(rng.integers(0, 2**63))
        h, s = oracle.hash_map(seed, m, d)
        S = oracle.materialize_S(h, s, d)
        # structure of Def. 1: every column of S has exactly one nonzero, equal to +-1
        nz = (S != 0).sum(axis=0)
        assert np.all(nz == 1) and np.all(np.abs(S[S != 0]) == 1.0)
        At, bt = oracle.sketch_dense(A, b, d, seed=seed)
        assert np.array_equal(At, oracle.dense_S_product(S, A))
        assert np.array_equal(bt, oracle.dense_S_product(S, b[:, None])[:, 0])


def test_sketch_spec_examples():
    """bucket (0,1,0), sign (+,-,+)."""
    A = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 7.0]])
    h = np.array([0, 1, 0], np.int32)
    s = np.array([1, -1, 1], np.int8)
    At, bt = oracle.sketch_dense(A, np.ones(3), 2, h=h, s=s)
    assert np.array_equal(At, np.array([[6.0, 9.0], [-3.0, -4.0]]))
    assert np.array_equal(bt, np.array([2.0, -1.0]))
    for i in range(3):                                # one-hot b -> sign * e_h
        e = np.zeros(3)
        e[i] = 1.0
        _, bt = oracle.sketch_dense(A, e, 2, h=h, s=s)
        want = np.zeros(2)
        want[h[i]] = s[i]
        assert np.array_equal(bt, want)
    At, bt = oracle.sketch_dense(np.zeros((3, 2)), np.zeros(3), 2, h=h, s=s)
    assert not At.any() and not bt.any()


def test_sketch_permutation_is_signed_row_permutation():
    """d = m with h a permutation -> signed row permutation of A."""
    rng = np.random.default_rng(5)
    m, n = 30, 4
    A = rng.standard_normal((m, n))
    perm = rng.permutation(m).astype(np.int32)
    s = rng.choice([-1, 1], m).astype(np.int8)
    At, _ = oracle.sketch_dense(A, np.zeros(m), m, h=perm, s=s)
    for i in range(m):
        assert np.array_equal(At[perm[i]], s[i] * A[i])


def test_sketch_column_sums_and_isometry_in_expectation():
    """sum_j A~[j,:] = sum_i s_i A[i,:] (Def. 1) and E||Sb||^2 = ||b||^2."""
    A, b, _ = _rng_problem(500, 6, 11)
    At, _ = oracle.sketch_dense(A, b, 37, seed=99)
    h, s = oracle.hash_map(99, 500, 37)
    lhs = At.sum(axis=0)
    rhs = (s[:, None] * A).sum(axis=0)
    bound = 2 * 500 * 2.0**-53 * np.abs(A).sum(axis=0) + 1e-300
    assert np.all(np.abs(lhs - rhs) <= bound)
    rng = np.random.default_rng(1)
    bvec = rng.standard_normal(64)
    ratios = []
    for seed in range(3000):
        _, bt = oracle.sketch_dense(np.zeros((64, 1)), bvec, 16, seed=seed)
        ratios.append(float(bt @ bt) / float(bvec @ bvec))
    ratios = np.array(ratios)
    assert abs(ratios.mean() - 1.0) < 5 * ratios.std() / np.sqrt(len(ratios))


def test_sketch_csr_equals_dense_of_same_matrix():
    rng = np.random.default_rng(8)
    m, n, d, k = 300, 40, 23, 5
    cols = np.sort(np.stack([rng.choice(n, k, replace=False) for _ in range(m)]), axis=1)
    vals = rng.standard_normal((m, k))
    A = np.zeros((m, n))
    for i in range(m):
        A[i, cols[i]] = vals[i]
    b = rng.standard_normal(m)
    rp = np.arange(m + 1, dtype=np.int64) * k
    At1, bt1 = oracle.sketch_csr(rp, cols.reshape(-1), vals.reshape(-1), b, n, d, seed=4)
    At2, bt2 = oracle.sketch_dense(A, b, d, seed=4)
    # dense adds +-0.0 for structural zeros; x + (+-0) == x, so the results are equal
    assert np.array_equal(At1, At2) and np.array_equal(bt1, bt2)


# ---------------------------------------------------------------- O-3 norms, residual
def test_row_norms_examples():
    """S:53-55."""
    assert np.array_equal(oracle.row_norms(np.eye(2)), [1.0, 1.0])
    assert np.array_equal(oracle.row_norms(np.array([[3.0, 4.0]])), [25.0])
    assert np.array_equal(oracle.row_norms(np.zeros((3, 4))), [0.0, 0.0, 0.0])
    A, _, _ = _rng_problem(40, 9, 2)
    nsq = oracle.row_norms(A)
    fro = float(np.linalg.norm(A, "fro")) ** 2
    assert abs(nsq.sum() - fro) <= 1e-13 * fro


def test_residual_example():
    """S:230's instance A = [[1,2],[3,4],[5,6]], b = A(1,1) = (3,7,11).  By hand:
    x = (1,0) gives b - Ax = (2,4,6) (S:230 prints (1,1,1), which is the value for
    x = (2,0); DESIGN.md §3 R-12 records the misprint), x = (2,0) gives (1,1,1)."""
    A = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    b = np.array([3.0, 7.0, 11.0])
    assert np.array_equal(oracle.residual(A, b, np.array([1.0, 0.0])), [2, 4, 6])
    assert np.array_equal(oracle.residual(A, b, np.array([2.0, 0.0])), [1, 1, 1])
    assert np.array_equal(oracle.residual(A, b, np.array([1.0, 1.0])), [0, 0, 0])


# ---------------------------------------------------------------- O-4 loop
def test_solve_identity_four_steps():
    """A = I4, b = (4,3,2,1): each step zeroes the largest coordinate -> 4 steps."""
    A = np.eye(4)
    b = np.array([4.0, 3.0, 2.0, 1.0])
    r = oracle.mwrk(A, b, x_star=b, tol=1e-30, trace=10)
    assert r.iterations == 4 and r.termination == oracle.CONVERGED
    assert r.idx_trace.tolist() == [0, 1, 2, 3]
    assert np.array_equal(r.x, b)


def test_solve_select_and_update_examples():
    """S:237-239 (selection, lowest-index ties) and S:248 (update)."""
    # r = (3,-4), nsq = (1,4): scores 9, 4 -> index 0
    r = oracle.solve(np.array([[1.0, 0.0], [0.0, 2.0]]), np.array([3.0, -4.0]),
                     np.array([1.0, 4.0]), x_star=np.array([3.0, -2.0]), max_iters=1, trace=1)
    assert r.idx_trace.tolist() == [0]
    # exact tie r = (2,2), nsq = (1,1) -> index 0
    r = oracle.solve(np.eye(2), np.array([2.0, 2.0]), np.ones(2), x_star=np.array([2.0, 2.0]),
                     max_iters=1, trace=1)
    assert r.idx_trace.tolist() == [0]
    # x = 0, row (3,4), b_i = 5 -> x = (0.6, 0.8)
    r = oracle.solve(np.array([[3.0, 4.0]]), np.array([5.0]), np.array([25.0]),
                     x_star=np.array([0.6, 0.8]), tol=1e-20)
    assert r.iterations == 1
    assert np.allclose(r.x, [0.6, 0.8], rtol=0, atol=2e-16)


def test_solve_zero_iterations_when_x0_is_solution():
    """S:282."""
    A, b, xs = _rng_problem(100, 5, 4)
    r = oracle.csk(A, b, 30, x0=xs, x_star=xs)
    assert r.iterations == 0 and r.termination == oracle.CONVERGED


def test_solve_n1_one_step():
    """n = 1: one projection lands on x* (closed form x = b_i / a_i)."""
    A, b, xs = _rng_problem(50, 1, 6)
    r = oracle.csk(A, b, 10, x_star=xs, tol=1e-20)
    assert r.iterations == 1
    assert abs(r.x[0] - xs[0]) <= 4 * 2.0**-53 * abs(xs[0])


def test_stagnated_masked_and_zero_sketch():
    # rank-deficient sketch: r = 0 on every row while RES > tol -> Stagnated
    r = oracle.solve(np.array([[1.0, 0.0]]), np.array([0.0]), np.array([1.0]),
                     x_star=np.array([0.0, 1.0]))
    assert r.termination == oracle.STAGNATED and r.iterations == 0
    # zero row with nonzero b~ is masked, never selected
    At = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    bt = np.array([100.0, 1.0, 2.0])
    r = oracle.solve(At, bt, oracle.row_norms(At), x_star=np.array([1.0, 2.0]), tol=1e-30,
                     trace=10)
    assert 0 not in r.idx_trace.tolist() and r.termination == oracle.CONVERGED
    with pytest.raises(ValueError):
        oracle.solve(np.zeros((2, 2)), np.ones(2), np.zeros(2), x_star=np.ones(2))


def test_csk_identity_map_reduces_to_mwrk_bitwise():
    """Remark 1: with d = m, h = id, any signs, CSK is MWRK; sign flips are exact."""
    A, b, xs = _rng_problem(60, 6, 9)
    s = np.random.default_rng(0).choice([-1, 1], 60).astype(np.int8)
    At, bt = oracle.sketch_dense(A, b, 60, h=np.arange(60, dtype=np.int32), s=s)
    r1 = oracle.solve(At, bt, oracle.row_norms(At), x_star=xs, tol=1e-12, trace=500)
    r2 = oracle.mwrk(A, b, x_star=xs, tol=1e-12, trace=500)
    assert r1.iterations == r2.iterations > 5
    assert np.array_equal(r1.idx_trace, r2.idx_trace)
    assert np.array_equal(r1.x, r2.x)


def _trajectory(m=2000, n=20, d=200, seed=17, kind="gauss"):
    A, b, xs = _rng_problem(m, n, seed, kind)
    At, bt = oracle.sketch_dense(A, b, d, seed=seed)
    nsq = oracle.row_norms(At)
    r = oracle.solve(At, bt, nsq, x_star=xs, tol=1e-14, trace=5000, trace_x=True)
    return A, At, bt, nsq, xs, r


def test_proof_identities_every_step():
    """eq:A, eq:5, eq:6, monotone, orthogonality."""
    A, At, bt, nsq, xs, r = _trajectory()
    assert r.termination == oracle.CONVERGED and r.iterations > 20
    fro = float(np.sum(At * At))
    spec2 = float(np.linalg.norm(At, 2)) ** 2
    n = At.shape[1]
    assert fro <= n * spec2 * (1 + 1e-12)                         # eq:6 last step
    for k, ik in enumerate(r.idx_trace):
        xk, xk1 = r.x_trace[k], r.x_trace[k + 1]
        e0, e1 = xk - xs, xk1 - xs
        E0, E1 = float(e0 @ e0), float(e1 @ e1)
        proj = float(At[ik] @ e0) ** 2 / nsq[ik]
        assert abs(E1 - (E0 - proj)) <= 1e-8 * E0                # eq:A
        res = bt - At @ xk
        mask = nsq > 0
        ratio = res[ik] ** 2 / nsq[ik]
        assert ratio >= (res[mask] @ res[mask]) / nsq[mask].sum() * (1 - 1e-12)   # eq:5
        assert np.all(res[mask] ** 2 / nsq[mask] <= ratio * (1 + 1e-12))         # argmax
        SAe = At @ e0
        assert E1 <= E0 - float(SAe @ SAe) / fro * (1 - 1e-9) + 1e-14 * E0       # eq:6 first
        assert np.sqrt(E1) <= np.sqrt(E0) * (1 + 1e-12)                           # monotone
        r_after = bt[ik] - At[ik] @ xk1
        scale = abs(bt[ik]) + np.sqrt(nsq[ik]) * np.linalg.norm(xk1)
        assert abs(r_after) <= 1e-9 * scale


def test_theorem2_rate_with_exact_distortion():
    """Theorem 2: per-step contraction 1 - (1-eps)^3 sigma_r^2 / (n ||A||^2)
    holds for every step once eps is the exact distortion of S on range(A)
    (both Lemma 1 inequalities then hold deterministically)."""
    m, n, d = 5000, 10, 400
    A, b, xs = _rng_problem(m, n, 21)
    seed = 5
    h, s = oracle.hash_map(seed, m, d)
    Q, _ = np.linalg.qr(A)
    SQ = np.zeros((d, n))
    np.add.at(SQ, h, s[:, None] * Q)
    sv = np.linalg.svd(SQ, compute_uv=False)
    eps = max(1 - sv.min() ** 2, sv.max() ** 2 - 1)
    assert 0 <= eps < 1
    svA = np.linalg.svd(A, compute_uv=False)
    rho = 1 - (1 - eps) ** 3 / n * svA.min() ** 2 / svA.max() ** 2
    At, bt = oracle.sketch_dense(A, b, d, seed=seed)
    r = oracle.solve(At, bt, oracle.row_norms(At), x_star=xs, tol=1e-20, max_iters=300,
                     trace=400, trace_x=True)
    E = [float((x - xs) @ (x - xs)) for x in r.x_trace]
    for k in range(len(E) - 1):
        if E[k] < 1e-24:
            break
        assert E[k + 1] <= rho * E[k] * (1 + 1e-9)


def test_scale_invariance_power_of_two():
    """scaling A and b by 2^e leaves the i_k sequence unchanged."""
    A, b, xs = _rng_problem(800, 12, 13)
    r1 = oracle.csk(A, b, 120, seed=1, x_star=xs, trace=3000)
    r2 = oracle.csk(A * 32.0, b * 32.0, 120, seed=1, x_star=xs, trace=3000)
    assert np.array_equal(r1.idx_trace, r2.idx_trace)


def test_residual_mode_converges():
    """Solution-free stop ||r||^2/||b~||^2 <= tol on a consistent system."""
    A, b, xs = _rng_problem(3000, 15, 23)
    r = oracle.csk(A, b, 150, seed=2, x_star=None, tol=1e-10)
    assert r.termination == oracle.CONVERGED
    At, bt = oracle.sketch_dense(A, b, 150, seed=2)
    rr = bt - At @ r.x
    assert float(rr @ rr) / float(bt @ bt) <= 1e-10 * (1 + 1e-6)
    # and the original system is solved too (x* solves both systems)
    assert np.linalg.norm(A @ r.x - b) / np.linalg.norm(b) <= 10 * np.sqrt(1e-10)


def test_max_iters_cap():
    A, b, xs = _rng_problem(2000, 30, 25)
    r = oracle.csk(A, b, 300, x_star=xs, tol=1e-6, max_iters=7)
    assert r.termination == oracle.MAX_ITERS and r.iterations == 7 and r.final_res > 1e-6


@pytest.mark.slow
def test_table1_iteration_means():
    """Table 1 at paper scale, d = n^2: the reading of Algorithm 1 reproduces
    the printed IT means (CSK within 3 %, MWRK within 2 iterations)."""
    rows = [[float(v) for v in t] for t in _golden_lines("table1_it.txt")]
    (m, n, d, csk_it, mwrk_it) = rows[0]
    m, n, d = int(m), int(n), int(d)
    its, mw = [], []
    for trial in range(10):
        g = torch.Generator().manual_seed(500 + trial)
        xs = torch.randn(n, generator=g, dtype=torch.float64).numpy()
        A = torch.randn(m, n, generator=g, dtype=torch.float64).numpy()
        b = A @ xs
        its.append(oracle.csk(A, b, d, seed=trial, x_star=xs, max_iters=20000).iterations)
        if trial < 6:
            mw.append(oracle.mwrk(A, b, x_star=xs, max_iters=20000).iterations)
    assert abs(np.mean(its) - csk_it) <= 0.03 * csk_it, its
    assert abs(np.mean(mw) - mwrk_it) <= 2.0, mw
    (m, n, d, csk_it, _) = rows[1]
    m, n, d = int(m), int(n), int(d)
    its = []
    for trial in range(5):
        g = torch.Generator().manual_seed(700 + trial)
        xs = torch.randn(n, generator=g, dtype=torch.float64).numpy()
        A = torch.randn(m, n, generator=g, dtype=torch.float64).numpy()
        its.append(oracle.csk(A, A @ xs, d, seed=trial, x_star=xs, max_iters=20000).iterations)
    assert abs(np.mean(its) - csk_it) <= 0.03 * csk_it, its

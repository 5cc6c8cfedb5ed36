"""Lemma 1 distortion and the Theorem 2 rate at the configs' sizes, on the GPU (SURVEY §8(f)
NEXT #4).  A verification tool, not a hot path: QR / SVD are library calls
(torch.linalg on cuSOLVER); the sketch of the orthonormal basis is libcsk's own kernel.

  eps11 = max(s_max(SQ)^2 - 1, 1 - s_min(SQ)^2), Q an orthonormal basis of range(A)   (eq. lem11)
  eps12 = max_i |s_i(A) / s_i(SA) - 1|                                                (eq. lem12)
  rho   = 1 - (1 - eps)^3 / n * s_r(A)^2 / ||A||_2^2                                   (Theorem 2)
  rho_M = 1 - s_r(A)^2 / max_i sum_{j != i} ||A^(j)||^2          (Remark 2: MWRK's factor)
and the largest observed one-step contraction ||x_{k+1} - x*||^2 / ||x_k - x*||^2 of the GPU
solve over its first `trace` iterations, which Theorem 2 bounds by rho (w.p. >= 1 - 2 delta).

python tools/distortion.py C1 C2 C3 300000x50 [--trace 400]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402


def problem(spec):
    if spec in CONFIGS:
        cfg = CONFIGS[spec]
        p = make_config(cfg, "cuda")
        return p.A, p.b, p.x_star, cfg.d, cfg.sketch_seed
    m, n = (int(v) for v in spec.split("x"))
    g = torch.Generator(device="cuda").manual_seed(m + n)
    xs = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    return A, A @ xs, xs, n * n, 0  # the paper's d = n^2


def main():
    trace = 400
    specs = []
    for a in sys.argv[1:]:
        if a.startswith("--trace"):
            trace = int(a.split("=")[1]) if "=" in a else trace
        else:
            specs.append(a)
    print("| problem | m x n, d | eps (lem11) | eps (lem12) | Theorem 2 rho (CSK) | Remark 2 rho (MWRK) | "
          "max observed contraction | iterations checked |")
    print("|---|---|---|---|---|---|---|---|")
    for spec in specs or ["C1", "C2", "C3"]:
        A, b, xs, d, seed = problem(spec)
        m, n = A.shape
        Q, R = torch.linalg.qr(A, mode="reduced")
        SQ, _, _ = csk.csk_sketch(Q.contiguous(), torch.zeros(m, dtype=torch.float64, device="cuda"), d, seed=seed)
        s = torch.linalg.svdvals(SQ)
        eps11 = max(float(s[0] ** 2 - 1.0), float(1.0 - s[-1] ** 2))
        At, bt, nsq = csk.csk_sketch(A, b, d, seed=seed)
        sA = torch.linalg.svdvals(R)  # the singular values of A
        sSA = torch.linalg.svdvals(At)
        eps12 = float((sA / sSA - 1.0).abs().max())
        eps = max(eps11, eps12)
        rho = 1.0 - (1.0 - eps) ** 3 / n * float(sA[-1] ** 2) / float(sA[0] ** 2)
        rn = (A * A).sum(dim=1)
        rho_m = 1.0 - float(sA[-1] ** 2) / float(rn.sum() - rn.min())  # max_i sum_{j != i} = total - min
        r = csk.csk_solve(At, bt, nsq, x_star=xs, trace=trace, trace_x=True)
        k = min(r.iterations, trace - 1)
        X = r.x_trace[: k + 1]
        e2 = ((X - xs[None, :]) ** 2).sum(dim=1)
        ratio = (e2[1:] / e2[:-1]).max().item() if k > 0 else float("nan")
        print(f"| {spec} | {m} x {n}, {d} | {eps11:.4f} | {eps12:.4f} | {rho:.8f} | {rho_m:.8f} | {ratio:.6f} "
              f"({'<=' if ratio <= rho else '>'} rho) | {k} |", flush=True)
        del A, Q, R, SQ, At


if __name__ == "__main__":
    main()

"""Paper-protocol reproduction of Table 1 on B200.

For every size m x n of Table 1: d = n^2, T trials of A, x* ~ randn, b = A x*, x0 = 0, stop at
RES <= 1e-6, cap 20 000.  CSK = csk_sketch (plan + sketch + norms) + csk_solve; MWRK =
csk_row_norms(A) + the same loop kernel on (A, b) (Remark 1).  Times are CUDA-event
milliseconds on the launching stream; the inputs are generated on the GPU (seeded) before the
timed region.  Printed beside the paper's means (tests/golden/table1_full.txt; the paper's CPU
column is MATLAB seconds on an unstated machine: context, not a target).

python tools/table1.py [--trials 50] [--sizes 300000x50,700000x150] [--json out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                      "table1_full.txt")
CAP = 20_000


def paper_rows():
    rows = {}
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        m, n, d, ci, mi, cc, mc = line.split()
        rows[(int(m), int(n))] = dict(d=int(d), csk_it=float(ci), mwrk_it=float(mi), csk_cpu=float(cc),
                                      mwrk_cpu=float(mc))
    return rows


def hbm_peak_gbs():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json), else the profiling guide's figure."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        for k in ("hbm_gbs_sustained", "hbm_gbs", "hbm_copy_gbs"):
            if k in pk:
                return float(pk[k])
    except (OSError, ValueError):
        pass
    return 6552.0


def trial_problem(m, n, trial):
    g = torch.Generator(device="cuda").manual_seed(1_000_003 * m + 7919 * n + trial)
    x_star = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    return A, A @ x_star, x_star


def run_size(m, n, d, trials, ctx):
    At = torch.empty(d, n, dtype=torch.float64, device="cuda")
    bt = torch.empty(d, dtype=torch.float64, device="cuda")
    nsq = torch.empty(d, dtype=torch.float64, device="cuda")
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    res = dict(csk_it=[], mwrk_it=[], csk_ms=[], mwrk_ms=[], csk_conv=0, mwrk_conv=0)
    for t in range(trials):
        A, b, xs = trial_problem(m, n, t)
        for warm in (True, False) if t == 0 else (False,):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            x.zero_()
            ev[0].record()
            csk.csk_sketch(A, b, d, seed=t, ctx=ctx, out=(At, bt, nsq))
            csk.csk_solve_async(At, bt, nsq, x, x_star=xs, tol=1e-6, max_iters=CAP, ctx=ctx)
            ev[1].record()
            rc = csk.csk_solve_wait(ctx)
            x.zero_()
            ev[2].record()
            nsq_a = csk.csk_row_norms(A, ctx=ctx)
            csk.csk_solve_async(A, b, nsq_a, x, x_star=xs, tol=1e-6, max_iters=CAP, ctx=ctx)
            ev[3].record()
            rm = csk.csk_solve_wait(ctx)
            torch.cuda.synchronize()
            if warm:
                continue
            res["csk_it"].append(rc.iterations)
            res["mwrk_it"].append(rm.iterations)
            res["csk_ms"].append(ev[0].elapsed_time(ev[1]))
            res["mwrk_ms"].append(ev[2].elapsed_time(ev[3]))
            res["csk_conv"] += int(rc.termination == csk.CONVERGED)
            res["mwrk_conv"] += int(rm.termination == csk.CONVERGED)
        del A, b, xs
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=50)
    ap.add_argument("--sizes", default="")
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    paper = paper_rows()
    sizes = sorted(paper) if not args.sizes else [tuple(int(v) for v in s.split("x")) for s in args.sizes.split(",")]
    ctx = csk.Context()
    out = []
    peak = hbm_peak_gbs()
    print("| m x n | d | IT CSK (paper) | IT MWRK (paper) | IT speedup (paper) | CSK ms | MWRK ms | "
          "MWRK GB/s | time speedup (paper CPU speedup) | vs HBM-bound MWRK | converged |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for (m, n) in sizes:
        pr = paper[(m, n)]
        r = run_size(m, n, pr["d"], args.trials, ctx)
        T = len(r["csk_it"])
        ci = sum(r["csk_it"]) / T
        mi = sum(r["mwrk_it"]) / T
        # times: the median over trials (the first measured trial of a size can include the one-off
        # capture of the plan's CUDA graph); iteration counts: the mean, as the paper reports them
        cm = sorted(r["csk_ms"])[T // 2]
        mm = sorted(r["mwrk_ms"])[T // 2]
        # MWRK reads all of A every iteration: its floor is IT x 8 m n / (measured HBM peak)
        gbs = 8.0 * m * n * mi / (mm * 1e-3) / 1e9
        floor_ms = mi * 8.0 * m * n / (peak * 1e9) * 1e3
        row = dict(m=m, n=n, d=pr["d"], trials=T, csk_it=ci, mwrk_it=mi, it_speedup=mi / ci, csk_ms=cm, mwrk_ms=mm,
                   time_speedup=mm / cm, mwrk_gbs=gbs, mwrk_hbm_floor_ms=floor_ms, speedup_vs_floor=floor_ms / cm,
                   csk_converged=r["csk_conv"], mwrk_converged=r["mwrk_conv"], paper=pr)
        out.append(row)
        print(f"| {m} x {n} | {pr['d']} | {ci:.2f} ({pr['csk_it']:.2f}) | {mi:.2f} ({pr['mwrk_it']:.2f}) | "
              f"{mi / ci:.4f} ({pr['mwrk_it'] / pr['csk_it']:.4f}) | {cm:.3f} | {mm:.3f} | {gbs:.0f} | "
              f"{mm / cm:.2f} ({pr['mwrk_cpu'] / pr['csk_cpu']:.2f}) | {floor_ms / cm:.2f} | "
              f"{r['csk_conv']}/{T}, {r['mwrk_conv']}/{T} |",
              flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

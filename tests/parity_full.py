"""Whole-trajectory parity of the full-size configs against the oracle (not part of the default
test run: the oracle needs minutes).  Writes the committed artifacts profiles/r02_parity_<cfg>.txt.

    python tests/parity_full.py C4 [--cap 50000]     # 8 GB dense A, 50k capped iterations
    python tests/parity_full.py C5                   # 4e6 x 2000 CSR, to RES <= 1e-6

What is compared (SURVEY.md §8(c) acceptance, north_star):
  * the sketch: the GPU's whole A~ and b~ against the oracle's fold of the same input bytes
    (bit-exact, ==);
  * the loop, free-running on both sides from x0 = 0 on the same A~ (the oracle's own row norms):
    termination, IT (within 5 % / both MaxIters), the i_k sequences (first divergence, if any),
    RES_k of every iteration (max relative difference), final RES (C4: within 1e-6 relative);
  * lockstep on the first iterations with the kernel's r_k trace (||r_gpu - r_orc|| <= 1e-10 ||r_orc||).
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402
from test_gpu_parity import _lockstep, _np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["C3", "C4", "C5"])
    ap.add_argument("--cap", type=int, default=0, help="iteration cap (default: the config's)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    cap = args.cap or cfg.max_iters
    out_path = args.out or os.path.join(ROOT, "profiles", f"r02_parity_{cfg.name}.txt")
    lines = []

    def log(s):
        print(s, flush=True)
        lines.append(s)

    log(f"# whole-trajectory parity, {cfg.name}: m={cfg.m} n={cfg.n} d={cfg.d} kind={cfg.kind} cap={cap} "
        f"tol={cfg.tol} (tests/parity_full.py)")
    t0 = time.time()
    p = make_config(cfg, "cuda")
    if cfg.kind == "csr":
        At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, cfg.n, cfg.d, seed=cfg.sketch_seed)
    else:
        At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
    g = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=cfg.tol, max_iters=cap, trace=cap + 1)
    K = 20
    gl = csk.csk_solve(At, bt, nsq, x_star=p.x_star, tol=1e-30, max_iters=K, trace=K + 1, trace_x=True,
                       trace_r=K + 1)
    torch.cuda.synchronize()
    log(f"gpu: IT={g.iterations} termination={['converged', 'max_iters', 'stagnated'][g.termination]} "
        f"final RES={g.final_res:.6e}  ({time.time() - t0:.1f} s incl. generation)")

    # ---- sketch: the whole A~ and b~ against the oracle fold of the same bytes
    t1 = time.time()
    if cfg.kind == "csr":
        At_o, bt_o = oracle.sketch_csr(_np(p.row_ptr), _np(p.col), _np(p.val), _np(p.b), cfg.n, cfg.d,
                                       seed=cfg.sketch_seed)
    else:
        At_o, bt_o = oracle.sketch_dense(_np(p.A), _np(p.b), cfg.d, seed=cfg.sketch_seed)
    Atn, btn, xs = _np(At), _np(bt), _np(p.x_star)
    del p
    torch.cuda.empty_cache()
    same_A = np.array_equal(Atn, At_o)
    same_b = np.array_equal(btn, bt_o)
    log(f"sketch: A~ bit-exact={same_A} b~ bit-exact={same_b} ({Atn.size} + {btn.size} values, "
        f"oracle {time.time() - t1:.1f} s)")
    nsq_o = oracle.row_norms(At_o)
    rel = np.abs(_np(nsq) - nsq_o) / np.where(nsq_o > 0, nsq_o, 1)
    log(f"nsq: max relative difference {rel.max():.3e}; bit-identical rows {int((_np(nsq) == nsq_o).sum())}/{cfg.d}")

    # ---- lockstep on the first K iterations with the r_k trace
    _lockstep(At, bt, nsq, gl.x_trace, gl.idx_trace, K, gl.r_trace)
    log(f"lockstep: first {K} iterations -- r_k within 1e-10 (normwise), same i_k, x_(k+1) within 1e-12: OK")

    # ---- free-running oracle on the same A~
    t2 = time.time()
    o = oracle.solve(At_o, bt_o, nsq_o, x_star=xs, tol=cfg.tol, max_iters=cap, trace=cap + 1)
    log(f"oracle: IT={o.iterations} termination={oracle.TERMINATION_NAMES[o.termination]} "
        f"final RES={o.final_res:.6e} ({time.time() - t2:.1f} s, 1 core)")
    gi, oi = _np(g.idx_trace), o.idx_trace
    n = min(len(gi), len(oi))
    diff = np.nonzero(gi[:n] != oi[:n])[0]
    log(f"i_k sequences: {n} compared, " + ("identical" if not len(diff) else
                                             f"first divergence at k={int(diff[0])} ({len(diff)} differ)"))
    gr, orr = _np(g.res_trace), o.res_trace
    nr = min(len(gr), len(orr))
    rr = np.abs(gr[:nr] - orr[:nr]) / orr[:nr]
    log(f"RES_k: {nr} iterations compared, max relative difference {rr.max():.3e}")
    ok_it = (g.termination == o.termination and
             abs(g.iterations - o.iterations) <= max(1, 0.05 * o.iterations))
    ok_res = (g.final_res <= cfg.tol and o.final_res <= cfg.tol) if o.termination == 0 else \
        abs(g.final_res - o.final_res) <= 1e-6 * o.final_res
    verdict = same_A and same_b and ok_it and ok_res and not len(diff)
    log(f"bar: termination equal and |IT_gpu - IT_orc| <= max(1, 5%): {ok_it}; "
        f"final RES {'<= tol for both' if o.termination == 0 else 'within 1e-6 relative'}: {ok_res}")
    log(f"PARITY {'PASS' if verdict else 'FAIL'} ({time.time() - t0:.0f} s total)")
    with open(out_path, "w") as f:
        f.write("\n".join(lines) + "\n")
    sys.exit(0 if verdict else 1)


if __name__ == "__main__":
    main()

"""Per-iteration time of the loop in both stop modes (x* known: RES on the iterate error; x*
unknown: RES on the sketched residual, P:180 / S:279) at the configs' sizes.

python tools/resmode_time.py C3 C4 C5 [--iters 300]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402


def sketch(cfg, p):
    if cfg.kind == "csr":
        return csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, p.n, cfg.d, seed=cfg.sketch_seed)
    return csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)


def main():
    iters = 300
    names = []
    for a in sys.argv[1:]:
        if a.startswith("--iters="):
            iters = int(a.split("=")[1])
        else:
            names.append(a)
    print("| config | stop mode | iterations | us / iteration | tiers |")
    print("|---|---|---|---|---|")
    for name in names or ["C3", "C4", "C5"]:
        cfg = CONFIGS[name]
        p = make_config(cfg, "cuda")
        At, bt, nsq = sketch(cfg, p)
        for mode, xs in (("x* (error)", p.x_star), ("residual", None)):
            best = None
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                r = csk.csk_solve(At, bt, nsq, x_star=xs, tol=1e-30, max_iters=iters)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) * 1e3 / max(r.iterations, 1)
                best = t if best is None else min(best, t)
            tiers = csk.csk_last_solve_tiers()
            print(f"| {name} | {mode} | {r.iterations} | {best:.2f} | G={tiers['num_ctas']} rr={tiers['reg_rows']} "
                  f"rt={tiers['tmem_rows']} rs={tiers['smem_rows']} ring={tiers['ring_stages']}x{tiers['ring_rows']} |",
                  flush=True)
        del At, bt, nsq, p
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

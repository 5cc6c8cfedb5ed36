"""Debug probe: per-phase cycle breakdown of the persistent solve kernel (CTA 0, warps 0/1).

python tools/phase_probe.py [C1 C2 C3 C4] [--ctas 148,74,16]
Phases: 0 GEMV+warp argmax, 1 barrier#1, 2 CTA reduce+publish, 3 poll, 4 combine+row fetch,
5 barrier#2, 6 update+RES.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

os.environ.setdefault("CSK_LIB", "prof")  # the phase profiler lives in libcsk_prof.so
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if a in CONFIGS] or ["C1", "C2", "C3"]
    ctas = [0]
    smem_modes = [0]
    css = [0]
    for a in sys.argv[1:]:
        if a.startswith("--ctas="):
            ctas = [int(v) for v in a.split("=")[1].split(",")]
        if a.startswith("--cs="):
            css = [int(v) for v in a.split("=")[1].split(",")]
        if a.startswith("--smem="):
            smem_modes = [int(v) for v in a.split("=")[1].split(",")]
    names_ph = ["gemv", "bar1", "final", "clus", "grid", "row", "bar2", "upd"]
    for nm in names:
        cfg = CONFIGS[nm]
        p = make_config(cfg, "cuda")
        At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
        cap = cfg.max_iters if nm != "C4" else 3000
        for G in ctas:
          for cs in css:
            for sm in smem_modes:
                ph = torch.zeros(32, dtype=torch.int64, device="cuda")
                csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, num_ctas=G, smem_rows=sm, cluster_size=cs, legacy=True)
                st = torch.cuda.Event(enable_timing=True)
                en = torch.cuda.Event(enable_timing=True)
                st.record()
                r = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, num_ctas=G, smem_rows=sm,
                                  cluster_size=cs, phase_cycles=ph, legacy=True)
                geo = csk.csk_last_solve_geometry()
                en.record()
                torch.cuda.synchronize()
                ms = st.elapsed_time(en)
                it = max(r.iterations, 1)
                c = ph.cpu().tolist()
                w0 = " ".join(f"{names_ph[i]}={c[i] / it / 1965:.2f}" for i in range(8))
                fine = ["cand", "dpush", "dpoll", "gpush", "gpoll", "rpoll", "rowpre", "rowupd"]
                w0 += " || " + " ".join(f"{fine[i]}={c[8 + i] / it / 1965:.2f}" for i in range(8))
                w1 = " ".join(f"{names_ph[i]}={c[16 + i] / it / 1965:.2f}" for i in range(8) if c[16 + i])
                print(f"{nm} G={geo['num_ctas']} CS={geo['cluster_size']} srows={geo['smem_rows']} IT={r.iterations} {ms * 1e3 / it:.2f} us/it | "
                      f"w0(us/it @1.965GHz): {w0} | w1: {w1}", flush=True)


if __name__ == "__main__":
    main()

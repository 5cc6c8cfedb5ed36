"""Debug probe: per-phase cycle breakdown of the default loop kernel (loop.cu, CTA 0, warps 0/1).

python tools/loop_probe.py [C1 C2 C3 C4] [--ctas=148,74]
Phases: 0 GEMV + group finalize, 1 B1 wait, 2 CTA argmax + publish, 3 spin, 4 TMA issue +
slot load, 5 B2 wait, 6 row wait, 7 update.  w0 = warp 0 (exchange), w7 = last warp (RES test).
"""
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

os.environ.setdefault("CSK_LIB", "prof")  # the phase profiler lives in libcsk_prof.so
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

NAMES = ["gemv+final", "arrive(leader)", "combine+publish", "spin", "post", "B2", "rowwait", "upd", "fence",
         "owner+tma", "stopchk", "owner", "sb+expect", "slotcp", "rowcp", "slot_reread_permille"]


def main():
    names = [a for a in sys.argv[1:] if a in CONFIGS or re.fullmatch(r"\d+x\d+", a)] or ["C1", "C2", "C3"]
    ctas = [0]
    wpgs = [0]
    for a in sys.argv[1:]:
        if a.startswith("--ctas="):
            ctas = [int(v) for v in a.split("=")[1].split(",")]
        if a.startswith("--wpg="):
            wpgs = [int(v) for v in a.split("=")[1].split(",")]
    for nm in names:
        if nm in CONFIGS:
            cfg = CONFIGS[nm]
            p = make_config(cfg, "cuda")
            At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
            cap = cfg.max_iters if nm != "C4" else 3000
        else:  # "DxN": a random A~ of that shape (b~ = A~ x*), 1500 iterations
            d, n = (int(v) for v in nm.split("x"))
            g = torch.Generator(device="cuda").manual_seed(d * 7919 + n)
            At = torch.randn(d, n, dtype=torch.float64, device="cuda", generator=g)
            xs = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
            bt, nsq, cap = At @ xs, (At * At).sum(1), 1500
            p = type("P", (), {"x_star": xs})()
        for G, wpg in [(g, w) for g in ctas for w in wpgs]:
            csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, num_ctas=G, group_warps=wpg)
            ph = torch.zeros(32 + 64 * 2 * 160, dtype=torch.int64, device="cuda")
            st = torch.cuda.Event(enable_timing=True)
            en = torch.cuda.Event(enable_timing=True)
            st.record()
            r = csk.csk_solve(At, bt, nsq, x_star=p.x_star, max_iters=cap, num_ctas=G, group_warps=wpg,
                              phase_cycles=ph)
            en.record()
            torch.cuda.synchronize()
            geo = csk.csk_last_solve_geometry()
            ms = st.elapsed_time(en)
            it = max(r.iterations, 1)
            c = ph.cpu().tolist()
            geoG = csk.csk_last_solve_geometry()["num_ctas"]
            sk = ph[32:32 + 64 * 2 * geoG].view(64, 2, geoG).cpu().double()
            if r.iterations > 72:
                pub, done = sk[:, 0, :], sk[:, 1, :]
                spread = (pub.max(1).values - pub.min(1).values).mean().item()
                lastpub_to_done = (done.min(1).values - pub.max(1).values).mean().item()
                done_spread = (done.max(1).values - done.min(1).values).mean().item()
                print(f"   skew (ns, mean over 64 iterations): publish spread {spread:.0f}, last publish -> first "
                      f"spin exit {lastpub_to_done:.0f}, spin-exit spread {done_spread:.0f}")
                late = (pub - pub.min(1, keepdim=True).values).mean(0)  # per CTA, ns after the first publish
                order = late.argsort(descending=True)[:6].tolist()
                q = [late[i * geoG // 4:(i + 1) * geoG // 4].mean().item() for i in range(4)]
                print("   latest publishers (CTA: mean ns after the first): "
                      + ", ".join(f"{i}: {late[i].item():.0f}" for i in order)
                      + f" | mean lateness by CTA quarter: {q[0]:.0f} {q[1]:.0f} {q[2]:.0f} {q[3]:.0f}"
                      + f" | median {late.median().item():.0f}")
            w0 = " ".join(f"{NAMES[i]}={c[i] / it:.0f}" for i in range(16))
            w7 = " ".join(f"{NAMES[i]}={c[16 + i] / it:.0f}" for i in range(16) if c[16 + i])
            print(f"{nm} G={geo['num_ctas']} wpg={wpg} IT={r.iterations} {ms * 1e3 / it:.2f} us/it = "
                  f"{ms * 1e6 / it * 1.965:.0f} cyc/it | w0 cyc/it: {w0} | w7: {w7}", flush=True)


if __name__ == "__main__":
    main()

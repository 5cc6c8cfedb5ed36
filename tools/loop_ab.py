"""A/B of the loop kernel across library builds: python tools/loop_ab.py lib1.so lib2.so ... [--configs C1,C3]
Each build runs in its own process (ctypes loads one libcsk per process): per config and stop mode,
the best of 5 of the loop's us/iteration (C4 capped at 5000 iterations, C5 at 300) and a hash of
the i_k trace (equal hashes = the same trajectory)."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(configs):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2004_02480_b200 as csk
    from csk_synth import CONFIGS, make_config
    out = {}
    for name in configs:
        cfg = CONFIGS[name]
        p = make_config(cfg, "cuda")
        if cfg.kind == "csr":
            At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, p.n, cfg.d, seed=cfg.sketch_seed)
        else:
            At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed)
        cap = {"C4": 5000, "C5": 300}.get(name, cfg.max_iters)
        for mode, xs in (("xstar", p.x_star), ("resid", None)):
            best, r = None, None
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                r = csk.csk_solve(At, bt, nsq, x_star=xs, tol=cfg.tol if xs is not None else 1e-12, max_iters=cap,
                                  trace=cap + 1)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) * 1e3 / max(r.iterations, 1)
                best = t if best is None else min(best, t)
            h = hashlib.sha1(r.idx_trace.cpu().numpy().tobytes()).hexdigest()[:10]
            out[f"{name}/{mode}"] = (round(best, 3), r.iterations, h)
        del At, bt, nsq, p
        torch.cuda.empty_cache()
    print("RESULT " + json.dumps(out), flush=True)


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2].split(","))
        return
    configs = "C1,C2,C3,C4,C5"
    libs = []
    for a in sys.argv[1:]:
        if a.startswith("--configs="):
            configs = a.split("=", 1)[1]
        else:
            path, sep, envs = a.partition(":")
            libs.append(os.path.abspath(path) + sep + envs)
    res = {}
    for lib in libs:
        path, _, envs = lib.partition(":")
        env = dict(os.environ, CSK_LIB=path)
        for kv in filter(None, envs.split(",")):
            k, v = kv.split("=", 1)
            env[k] = v
        o = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", configs], env=env,
                           capture_output=True, text=True)
        line = [x for x in o.stdout.splitlines() if x.startswith("RESULT ")]
        if not line:
            print(f"{lib}: FAILED\n{o.stderr[-3000:]}", flush=True)
            continue
        res[lib] = json.loads(line[0][7:])
    keys = sorted({k for r in res.values() for k in r})
    print("| config/mode | " + " | ".join(os.path.basename(x) for x in res) + " |")
    print("|---|" + "---|" * len(res))
    for k in keys:
        cells = []
        for lib in res:
            v = res[lib].get(k)
            cells.append("-" if v is None else f"{v[0]} us (IT {v[1]}, {v[2]})")
        print(f"| {k} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()

import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2004_02480_b200 as csk
from csk_synth import CONFIGS, make_config
for nm in sys.argv[1:]:
    cfg = CONFIGS[nm]; p = make_config(cfg, "cuda")
    At = torch.empty(cfg.d, cfg.n, dtype=torch.float64, device="cuda"); bt = torch.empty(cfg.d, dtype=torch.float64, device="cuda"); nsq = torch.empty_like(bt)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ts = []
    for k in range(8):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed, out=(At, bt, nsq)); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(nm, os.environ.get("CSK_PLAN_CUB", "scan"), "sketch ms median", sorted(ts[2:])[len(ts[2:]) // 2])

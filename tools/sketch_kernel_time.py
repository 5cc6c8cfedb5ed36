"""Sketch kernel time alone (libcsk kernel events): python tools/sketch_kernel_time.py C3 300000x300 ...
(m x n specs use d = 10 n).  Env toggles (CSK_WPB_MAX_N, CSK_SKETCH_NO_WPB) pick the kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

ctx = csk.Context()
csk.csk_ctx_set_timing(True, ctx=ctx)
tag = os.environ.get("CSK_WPB_MAX_N", "default")
for spec in sys.argv[1:]:
    if spec in CONFIGS:
        cfg = CONFIGS[spec]
        p = make_config(cfg, "cuda")
        A, b, d, m, n = p.A, p.b, cfg.d, cfg.m, cfg.n
    else:
        m, n = (int(v) for v in spec.split("x"))
        d = 10 * n
        A = torch.randn(m, n, dtype=torch.float64, device="cuda")
        b = torch.randn(m, dtype=torch.float64, device="cuda")
    ks = []
    for _ in range(5):
        csk.csk_sketch(A, b, d, seed=1, ctx=ctx)
        torch.cuda.synchronize()
        ks.append(csk.csk_last_kernel_ms("sketch", ctx=ctx))
    k = sorted(ks)[2]
    print(f"{spec} n={n} wpb_max={tag}: kernel {k * 1e3:.1f} us = {8 * m * n / (k * 1e-3) / 1e9:.0f} GB/s", flush=True)
    del A, b

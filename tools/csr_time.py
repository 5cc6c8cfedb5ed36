"""CSR sketch kernel time (C5 and smaller): python tools/csr_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

cfg = CONFIGS["C5"]
p = make_config(cfg, "cuda")
nnz = int(p.row_ptr[-1].item())
for _ in range(4):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, cfg.n, cfg.d, seed=cfg.sketch_seed)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    by = 12 * nnz + 16 * (cfg.m + 1) + 8 * cfg.m + 8 * cfg.d * cfg.n + 16 * cfg.d
    print(f"C5 csk_sketch_csr {ms:.3f} ms  ({by / 1e6:.0f} MB algorithmic, {by / (ms * 1e-3) / 1e9:.0f} GB/s)", flush=True)
    del At, bt, nsq

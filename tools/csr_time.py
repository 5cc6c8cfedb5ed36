"""CSR sketch time at C5: the whole csk_sketch_csr call (plan + kernel) and the kernel alone
(libcsk's CUDA events, csk_ctx_set_timing): python tools/csr_time.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402
from csk_synth import CONFIGS, make_config  # noqa: E402

cfg = CONFIGS["C5"]
p = make_config(cfg, "cuda")
nnz = int(p.row_ptr[-1].item())
ctx = csk.Context()
csk.csk_ctx_set_timing(True, ctx=ctx)
by = 12 * nnz + 8 * (cfg.m + 1) + 8 * cfg.m + 8 * cfg.d * cfg.n + 16 * cfg.d
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    flush.fill_(1.0)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, cfg.n, cfg.d, seed=cfg.sketch_seed, ctx=ctx)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    kms = csk.csk_last_kernel_ms("sketch", ctx=ctx)
    print(f"C5 csk_sketch_csr {ms:.3f} ms ({by / (ms * 1e-3) / 1e9:.0f} GB/s), kernel {kms:.3f} ms "
          f"({by / (kms * 1e-3) / 1e9:.0f} GB/s of {by / 1e6:.0f} MB algorithmic)", flush=True)
    del At, bt, nsq

"""Is the dense sketch bound by random row gathers?  The same kernel (k_sketch_dense_wpb for n <= 256,
k_sketch_dense above: C3 and C4 shapes too)
with a random map (the hash) and with a monotone map (bucket j = rows [j m/d, (j+1) m/d): the
rows are read in address order).  python tools/gather_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402

ctx = csk.Context()
csk.csk_ctx_set_timing(True, ctx=ctx)
for m, n, d in [(700000, 50, 2500), (700000, 100, 10000), (700000, 150, 22500), (100000, 500, 5000),
                (1000000, 1000, 10000)]:
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    b = torch.randn(m, dtype=torch.float64, device="cuda")
    h_rand, s_rand = csk.csk_hash(m, d, seed=3)
    h_mono = (torch.arange(m, device="cuda", dtype=torch.int64) * d // m).to(torch.int32)
    for name, h, s in [("random", h_rand, s_rand), ("monotone", h_mono, s_rand)]:
        ks = []
        for _ in range(4):
            csk.csk_sketch_with_map(A, b, d, h, s, ctx=ctx)
            torch.cuda.synchronize()
            ks.append(csk.csk_last_kernel_ms("sketch", ctx=ctx))
        k = sorted(ks)[1]
        print(f"{m}x{n} d={d} {name}: kernel {k * 1e3:.1f} us = {8 * m * n / (k * 1e-3) / 1e9:.0f} GB/s", flush=True)

"""S4 (exact-order row norms) kernel time at the configs' A~ shapes, after an L2 flush:
python tools/norms_time.py   (CSK_NORMS_PLAIN=1: the thread-loaded kernel, for A/B)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
tag = "plain" if os.environ.get("CSK_NORMS_PLAIN") else "tma"
for name, d, n in [("C3", 5000, 500), ("C4", 10000, 1000), ("C5", 40000, 2000)]:
    At = torch.randn(d, n, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(6):
        flush.fill_(1.0)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        nsq = csk.csk_row_norms(At)
        en.record()
        torch.cuda.synchronize()
        ts.append(st.elapsed_time(en))
    ms = sorted(ts[1:])[len(ts[1:]) // 2]
    print(f"{tag:5s} {name} d={d} n={n}: {ms * 1e3:.1f} us ({8 * d * n / (ms * 1e-3) / 1e9:.0f} GB/s)", flush=True)
    del At

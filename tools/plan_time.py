"""Time csk_plan (S1+S2) alone: python tools/plan_time.py  (CSK_PLAN_CUB=1: the CUB radix path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_02480_b200 as csk  # noqa: E402

for m, d in [(1000, 500), (20000, 2000), (100000, 5000), (300000, 2500), (700000, 22500), (1000000, 10000),
             (4000000, 40000)]:
    ts = []
    for k in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        csk.csk_plan(m, d, seed=5)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"plan m={m} d={d} {'cub' if os.environ.get('CSK_PLAN_CUB') else 'fused'}: "
          f"{sorted(ts[1:])[2] * 1e3:.1f} us", flush=True)

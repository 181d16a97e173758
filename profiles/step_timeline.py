"""Kernel timeline of planned n=16384 steps (torch.profiler / CUPTI): per-kernel durations
and the gaps between consecutive kernels, to account for step time beyond GEMM + packs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
pl = mh.Plan(mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n)), mh.OP_SUB)
for _ in range(5):
    pl.run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(6):
        pl.run()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
prev_end = None
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    gap = (st - prev_end) if prev_end is not None else 0
    print(f"{e.name[:40]:40s} start {st:12.1f} us  dur {en - st:9.1f} us  gap {gap:7.1f} us")
    prev_end = max(prev_end or 0, en)

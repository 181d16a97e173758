"""Kernel timeline (torch.profiler / CUPTI) of planned steps of a BASELINE shape:
per-kernel durations and gaps.  python profiles/step_timeline_cfg.py [cfg3|cfg2|cfg1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
q = 65521
if which == "cfg3":
    n, t, oi, oj, r, k, c, op = 8192, 64, 96, 160, 6144, 2048, 5120, mh.OP_SUB
elif which == "cfg2":
    n, t, oi, oj, r, k, c, op = 4096, 64, 0, 0, 4096, 4096, 4096, mh.OP_SUB
else:
    n, t, oi, oj, r, k, c, op = 512, 32, 0, 0, 512, 512, 512, mh.OP_SET
lay, mod = mh.Layout(n, t), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
z = mh.encode(lay, oi, oj)
pl = mh.Plan(mh.Problem(mh.Sub(A, z, r, c), mh.Sub(B, z, r, k), mh.Sub(C, z, k, c)), op)
for _ in range(5):
    pl.run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(4):
        pl.run()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
prev_end = None
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    gap = (st - prev_end) if prev_end is not None else 0
    print(f"{e.name[:40]:40s} start {st:12.1f} us  dur {en - st:9.1f} us  gap {gap:7.1f} us")
    prev_end = max(prev_end or 0, en)

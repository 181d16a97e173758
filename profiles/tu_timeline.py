"""CUPTI kernel timeline of one TU sweep (n = 16384, panel 1024, p = 65521): per step the pack
and GEMM durations, the gaps, and the GEMM's time per tile wave (tiles / 148 rounded up).
  python profiles/tu_timeline.py [n] [block]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402
from paper_1705_04807_b200.tu import schur_plans, schur_sweep  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
block = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
q = 65521
f = torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda")
M = mh.Matrix.wrap(mh.Layout(n, 64), mh.Modulus(q), f.data_ptr(), owner=f)
plans = schur_plans(M, block)
for _ in range(2):
    schur_sweep(M, block, plans=plans)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    schur_sweep(M, block, plans=plans)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev = t0
k = 0
tot_g = 0.0
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    name = "gemm" if "k_gemm" in e.name else ("pack" if "pack" in e.name else e.name[:20])
    line = f"{name:5s} dur {en - st:8.1f} us gap {st - prev:6.1f} us"
    if name == "gemm":
        m = n - block * (k + 1)
        tiles = math.ceil(m / 128) ** 2
        waves = math.ceil(tiles / 148)
        macs = m * m * block
        line += f"  m={m:5d} tiles={tiles:5d} waves={waves:3d} us/wave={(en - st) / waves:6.2f} rate={macs / ((en - st) * 1e-6):.3e}"
        tot_g += en - st
        k += 1
    print(line)
    prev = en
span = evs[-1].time_range.end - t0
macs = sum((n - b) ** 2 * block for b in range(block, n, block))
print(f"sweep span {span / 1e3:.3f} ms ({macs / (span * 1e-6):.3e} GF(p) MAC/s), GEMMs {tot_g / 1e3:.3f} ms")

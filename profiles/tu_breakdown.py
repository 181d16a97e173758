"""Per-step breakdown of the TU sweep: full planned step (pack lhs + pack rhs +
GEMM) vs the GEMM kernel alone, and each step's GF(p) MAC/s.
  python profiles/tu_breakdown.py [n] [block]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402
from paper_1705_04807_b200.tu import schur_plans  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
block = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
q = 65521
f = torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda")
M = mh.Matrix.wrap(mh.Layout(n, 64), mh.Modulus(q), f.data_ptr(), owner=f)
plans = schur_plans(M, block)
tot_step = tot_gemm = tot_macs = 0.0
for i, pl in enumerate(plans):
    for _ in range(2):
        pl.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pl.run()
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 5
    g = pl.time_gemm(5)
    macs = pl.counters().scalar_macs
    tot_step += step
    tot_gemm += g
    tot_macs += macs
    rest = n - block * (i + 1)
    print(f"step {i:2d} {rest:5d}^2 x {block}: step {step:.3f} ms  gemm {g:.3f} ms  "
          f"({macs / g / 1e9:.3e} MAC/s gemm, {macs / step / 1e9:.3e} step)", flush=True)
print(f"TOTAL step {tot_step:.2f} ms gemm {tot_gemm:.2f} ms  overhead {tot_step - tot_gemm:.2f} ms  "
      f"{tot_macs / tot_step / 1e9 * 1e3:.3e} MAC/s")

"""GEMM-only rate against the inner length K (the TU regime is short K): Schur views
15360 x K x 15360 at (1024, 1024) of n = 16384 containers, p = 65521, C -= A.B, medians of 5
(plan.time_gemm), with the limb-adjusted roofline fraction (2 x measured bf16 burst / L^2).

  python profiles/k_curve.py
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    bf16 = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
except Exception:
    bf16 = 1590.0
roof = 2 * bf16 * 1e12 / 2 / 4  # int8 MAC/s / L^2, L = 2
n, q, m = 16384, 65521, 15360
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
z = mh.encode(lay, 1024, 1024)
print(f"# roofline {roof:.3e} GF(p) MAC/s (2 x {bf16} TFLOP/s bf16 burst, L = 2)")
for K in (128, 256, 512, 1024, 1536, 2048, 3072, 4096, 8192, 15360):
    plan = mh.Plan(mh.Problem(mh.Sub(A, z, m, m), mh.Sub(B, z, m, K), mh.Sub(C, z, K, m)), mh.OP_SUB)
    plan.run()
    torch.cuda.synchronize()
    ms = statistics.median(plan.time_gemm(5) for _ in range(5))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        plan.run()
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 5
    rate = m * m * K / (ms * 1e-3)
    print(f"K={K:6d}  GEMM {ms:8.3f} ms  {rate:.3e} GF(p) MAC/s  frac {rate / roof:.2f}   "
          f"step (packs + GEMM) {step:8.3f} ms  {m * m * K / (step * 1e-3):.3e}", flush=True)
    del plan

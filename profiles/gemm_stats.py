"""Diagnostics: per-CTA wait-cycle shares of k_gemm (MHG_GEMM_STATS=1) for a
few workloads.  Usage (GPU): MHG_GEMM_STATS=1 python profiles/gemm_stats.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

for (n, t, q, op) in [(16384, 64, 65521, mh.OP_SUB), (8192, 64, 2147483647, mh.OP_SET),
                      (4096, 64, 65521, mh.OP_SUB)]:
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
    A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
    prob = mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n))
    for _ in range(3):
        mh.mm(prob, op)
    torch.cuda.synchronize()
    print(f"n={n} q={q}", flush=True)

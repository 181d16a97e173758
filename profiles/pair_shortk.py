"""Single-CTA k_gemm vs CTA-pair k_gemm2 (MHG_OPT_GEMM_KERNEL 1 / 2) on the short-K Schur
views (15360 x K x 15360 at (1024, 1024), n = 16384, p = 65521, C -= A.B), interleaved.
python profiles/pair_shortk.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
z = mh.encode(lay, 1024, 1024)
for K in (1024, 2048, 4096, 15360):
    prob = mh.Problem(mh.Sub(A, z, 15360, 15360), mh.Sub(B, z, 15360, K), mh.Sub(C, z, K, 15360))
    plans = {}
    for name, kern in (("1cta", 1), ("pair", 2)):
        with mh.options({mh.OPT_GEMM_KERNEL: kern}):
            plans[name] = mh.Plan(prob, mh.OP_SUB)
        plans[name].run()
    res = {k: [] for k in plans}
    for _ in range(3):
        for name, pl in plans.items():
            res[name].append(pl.time_gemm(5))
    print(f"K={K}: " + "  ".join(f"{k} {statistics.median(v):.3f} ms" for k, v in res.items()), flush=True)

"""K = 1024 Schur-view GEMM (15360 x 1024 x 15360 at (1024, 1024), n = 16384) timed for
C -= A.B and C = A.B (no C_old read) and at K = 2048 / 4096: how much of the short-K tile
time the C_old path costs.  python profiles/shortk_ops.py"""
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
for K in (1024, 2048, 4096):
    prob = mh.Problem(mh.Sub(A, z, 15360, 15360), mh.Sub(B, z, 15360, K), mh.Sub(C, z, K, 15360))
    res = {}
    for name, op in (("sub", mh.OP_SUB), ("set", mh.OP_SET), ("add", mh.OP_ADD)):
        pl = mh.Plan(prob, op)
        pl.run()
        res[name] = statistics.median(pl.time_gemm(5) for _ in range(5))
    macs = 15360 * 15360 * K
    print(f"K={K}: " + "  ".join(f"{k} {v:.3f} ms ({macs / v / 1e9:.3e} MAC/s)" for k, v in res.items()),
          flush=True)

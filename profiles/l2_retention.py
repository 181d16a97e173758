"""One-group GEMM (M = 1024 = 8 row tiles, N = K = 16384): the group's 8 lhs panels (32 MB)
are re-used by all ~7 waves.  DRAM read ~0.68 GB if they stay in L2, ~0.87 GB if each wave
re-reads them.  Run under ncu --metrics dram__bytes_read.sum -k regex:k_gemm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
for spec in sys.argv[1:] or ["MHG_DUMMY=0"]:
    k, v = spec.split("=", 1)
    os.environ[k] = v
    pl = mh.Plan(mh.Problem(mh.Sub(A, 0, 1024, n), mh.Sub(B, 0, 1024, n), mh.Sub(C, 0, n, n)), mh.OP_SUB)
    pl.run()
    torch.cuda.synchronize()
    print(spec, pl.time_gemm(1), flush=True)
    del os.environ[k]

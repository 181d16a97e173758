"""One n=16384 GEMM launch per env variant, for ncu DRAM-byte comparisons:
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \\
      -k regex:k_gemm python profiles/l2_traffic.py VAR=VAL ...
Each variant: plan created + run once (packs filled) + time_gemm(1) inside its env."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
prob = mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n))
for spec in sys.argv[1:] or ["MHG_DUMMY=0"]:
    k, v = spec.split("=", 1)
    os.environ[k] = v
    pl = mh.Plan(prob, mh.OP_SUB)
    pl.run()
    torch.cuda.synchronize()
    ms = pl.time_gemm(1)
    print(f"{spec}: {ms:.3f} ms", flush=True)
    del os.environ[k]
    del pl

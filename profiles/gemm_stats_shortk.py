"""MHG_GEMM_STATS=1 diagnostics for short-K updates (cfg3 shape, K=1024 TU step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1705_04807_b200 as mh
q = 65521
for (n, oi, oj, r, k, c) in [(8192, 96, 160, 6144, 2048, 5120), (16384, 1024, 1024, 15360, 1024, 15360),
                             (16384, 0, 0, 16384, 4096, 16384)]:
    lay, mod = mh.Layout(n, 64), mh.Modulus(q)
    fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
    A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
    z = mh.encode(lay, oi, oj)
    prob = mh.Problem(mh.Sub(A, z, r, c), mh.Sub(B, z, r, k), mh.Sub(C, z, k, c))
    for _ in range(2):
        mh.mm(prob, mh.OP_SUB)
    torch.cuda.synchronize()
    print(f"n={n} view {r}x{k}x{c}", flush=True)
    del A, B, C, fl; torch.cuda.empty_cache()

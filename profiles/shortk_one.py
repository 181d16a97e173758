"""One short-K Schur update (n=16384, 15360 x K x 15360 view, K=1024) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1705_04807_b200 as mh
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
z = mh.encode(lay, 1024, 1024)
prob = mh.Problem(mh.Sub(A, z, 15360, 15360), mh.Sub(B, z, 15360, K), mh.Sub(C, z, K, 15360))
for _ in range(3):
    mh.mm(prob, mh.OP_SUB)
torch.cuda.synchronize()
print("done")

"""Pack-kernel share of a planned step: step time (events) minus the GEMM
time bracketed by the plan's profiling events.  Usage: python profiles/pack_time.py [n] [q]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1705_04807_b200 as mh
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = int(sys.argv[2]) if len(sys.argv) > 2 else 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
for name, (r0, c0, rr, kk, cc) in {"full": (0, 0, n, n, n), "misaligned": (96, 160, n - 256, n - 512, n - 384)}.items():
    pl = mh.Plan(mh.Problem(mh.Sub(A, mh.encode(lay, r0, c0), rr, cc), mh.Sub(B, mh.encode(lay, r0, c0), rr, kk),
                            mh.Sub(C, mh.encode(lay, r0, c0), kk, cc)), mh.OP_SUB)
    pl.set_profiling(True)
    for _ in range(3):
        pl.run()
    torch.cuda.synchronize(); pl.gemm_time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        pl.run()
    e1.record(); torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 20
    g, cnt = pl.gemm_time()
    g /= cnt
    pack = step - g
    L = mh.limb_params(q)[0]
    byts = (rr * kk + kk * cc) * (4 + L)
    print(f"{name:11s} n={n} step {step:.3f} ms gemm {g:.3f} ms pack(lhs+rhs) {pack:.3f} ms "
          f"= {byts / pack / 1e6:.0f} GB/s of algorithmic bytes", flush=True)

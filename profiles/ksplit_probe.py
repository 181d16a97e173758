"""Would splitting a very long K into two chained multiplies (panels half as long, so the
wave's operand panels sit in L2 better) pay at n = 32768?  One K = 32768 plan against two
K = 16384 plans on column / row halves of the same operands (C -= A1 B1; C -= A2 B2).

  python profiles/ksplit_probe.py [n]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q = 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
C, A, B = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
h = n // 2
full = mh.Plan(mh.Problem(mh.Sub(C, 0, n, n), mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n)), mh.OP_SUB)
halves = [mh.Plan(mh.Problem(mh.Sub(C, 0, n, n), mh.Sub(A, mh.encode(lay, 0, k0), n, h),
                             mh.Sub(B, mh.encode(lay, k0, 0), h, n)), mh.OP_SUB) for k0 in (0, h)]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for rnd in range(3):
    t_full = timed(lambda: full.run(), 5)
    t_half = timed(lambda: [p.run() for p in halves], 5)
    g_full = statistics.median(full.time_gemm(2) for _ in range(3))
    g_half = sum(statistics.median(p.time_gemm(2) for _ in range(3)) for p in halves)
    print(f"n={n} round {rnd}: one plan {t_full:.2f} ms (GEMM {g_full:.2f})   two K-halves {t_half:.2f} ms "
          f"(GEMMs {g_half:.2f})   ratio {t_half / t_full:.4f}", flush=True)

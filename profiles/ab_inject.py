"""C_old injection A/B at the step level (planned pack(A) + pack(B) [+ pack(C_old)]
+ GEMM, CUDA events on the launching stream), short-K Schur updates
C(15360 x 15360) -= A(15360 x K) B(K x 15360) inside n = 16384 parents at (1024, 1024),
p = 65521.  Variants interleaved, median of AB_ROUNDS rounds of 10 runs.

  python profiles/ab_inject.py [K ...]
"""
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
Ks = [int(x) for x in sys.argv[1:]] or [256, 512, 768, 1024, 1536, 2048, 3072]
s = torch.cuda.Stream()
rounds = int(os.environ.get("AB_ROUNDS", "5"))
for K in Ks:
    prob = mh.Problem(mh.Sub(A, z, 15360, 15360), mh.Sub(B, z, 15360, K), mh.Sub(C, z, K, 15360))
    plans = {}
    for name, kt in (("load", "0"), ("inject", "1000")):
        os.environ["MHG_INJECT_KT"] = kt
        plans[name] = mh.Plan(prob, mh.OP_SUB)
    times = {k: [] for k in plans}
    for _ in range(rounds):
        for name, pl in plans.items():
            pl.run(s)
            b, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b.record(s)
            for _ in range(10):
                pl.run(s)
            e.record(s)
            e.synchronize()
            times[name].append(b.elapsed_time(e) / 10)
    macs = 15360 * 15360 * K
    line = " ".join(f"{k}={statistics.median(v):.3f}ms ({macs / statistics.median(v) / 1e9:.3g} MAC/s)"
                    for k, v in times.items())
    print(f"K={K}: {line}  speedup={statistics.median(times['load']) / statistics.median(times['inject']):.3f}",
          flush=True)

"""Short-K GEMM kernels A/B in one process: MHG_OPT_GEMM_KERNEL variants on the Schur views
15360 x K x 15360 at (1024, 1024) of n = 16384 (p = 65521, C -= A.B), GEMM-only median of
5 x plan.time_gemm(5), plus the TU sweep (panel 1024) per variant.
  python profiles/ab_kernels_shortk.py [rounds] name=VALUE ...   (e.g. 1cta=1 pair=2)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402
from paper_1705_04807_b200.tu import schur_plans, schur_sweep  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
variants = [(a.split("=")[0], int(a.split("=")[1])) for a in sys.argv[1:] if "=" in a] or [("1cta", 1), ("pair", 2)]
rounds = int(args[0]) if args else 2
Ks = [int(k) for k in os.environ.get("AB_KS", "512,1024,2048,4096,8192").split(",")]
n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
z = mh.encode(lay, 1024, 1024)
plans = {}
for name, v in variants:
    with mh.options({mh.OPT_GEMM_KERNEL: v}):
        for K in Ks:
            pl = mh.Plan(mh.Problem(mh.Sub(A, z, 15360, 15360), mh.Sub(B, z, 15360, K), mh.Sub(C, z, K, 15360)), mh.OP_SUB)
            pl.run()
            plans[(name, K)] = pl
        plans[(name, "tu")] = schur_plans(A, 1024)
        schur_sweep(A, 1024, plans=plans[(name, "tu")])
torch.cuda.synchronize()
for r in range(rounds):
    for name, v in variants:
        out = {}
        for K in Ks:
            pl = plans[(name, K)]
            ms = statistics.median(pl.time_gemm(5) for _ in range(5))
            out[f"K{K}"] = round(ms, 4)
            out[f"K{K}_macs"] = f"{15360 * 15360 * K / (ms * 1e-3):.3e}"
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); macs = schur_sweep(A, 1024, plans=plans[(name, "tu")]); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out["tu1024_ms"] = round(statistics.median(ts), 3)
        out["tu1024_macs"] = f"{macs / (statistics.median(ts) * 1e-3):.3e}"
        print(f"round {r} {name:6s} {out}", flush=True)

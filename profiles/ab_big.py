"""A/B of library builds on the n = 32768 cfg5 GEMM (C -= A.B, 32768^3): one process per
build, builds interleaved, median of 3 x time_gemm(2).
  python profiles/ab_big.py r1=variants/libmhg_r1.so new=paper_1705_04807_b200/libmhg.so"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, statistics, sys
sys.path.insert(0, os.environ["AB_ROOT"])
import torch
import paper_1705_04807_b200 as mh
n, q = 32768, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
plan = mh.Plan(mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n)), mh.OP_SUB)
plan.run()
print("%.2f ms" % statistics.median(plan.time_gemm(2) for _ in range(3)))
'''
for r in range(int(os.environ.get("AB_ROUNDS", "2"))):
    for name, lib in (a.split("=", 1) for a in sys.argv[1:]):
        env = dict(os.environ, MHG_LIB=os.path.join(ROOT, lib), AB_ROOT=ROOT)
        res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(f"round {r} {name:8s} {res.stdout.strip() or res.stderr[-300:]}", flush=True)

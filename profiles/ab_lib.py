"""A/B of library builds (MHG_LIB=variants/libmhg_<name>.so, one process per build, ABAB
order) on short- and long-K Schur views of n = 16384 (15360 x K x 15360 at (1024, 1024))
plus the TU sweep (panel 1024).  Prints one line per (build, round).

  python profiles/ab_lib.py base=paper_1705_04807_b200/libmhg.so pf=variants/libmhg_pf.so
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, statistics, sys
sys.path.insert(0, os.environ["AB_ROOT"])
import torch
import paper_1705_04807_b200 as mh
from paper_1705_04807_b200.tu import schur_plans, schur_sweep
n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
z = mh.encode(lay, 1024, 1024)
out = {}
for K in [int(k) for k in os.environ.get("AB_KS", "1024,2048,4096,15360").split(",")]:
    plan = mh.Plan(mh.Problem(mh.Sub(A, z, 15360, 15360), mh.Sub(B, z, 15360, K), mh.Sub(C, z, K, 15360)), mh.OP_SUB)
    plan.run()
    out[f"K{K}"] = statistics.median(plan.time_gemm(5) for _ in range(5))
    del plan
plan = mh.Plan(mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n)), mh.OP_SUB)
plan.run()
out["ns16k"] = statistics.median(plan.time_gemm(3) for _ in range(5))
del plan
M = A
plans = schur_plans(M, 1024)
schur_sweep(M, 1024, plans=plans)
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); macs = schur_sweep(M, 1024, plans=plans); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
out["tu1024_ms"] = statistics.median(ts)
out["tu1024_macs"] = macs / (out["tu1024_ms"] * 1e-3)
print(json.dumps(out))
'''

variants = [a.split("=", 1) for a in sys.argv[1:]]
rounds = int(os.environ.get("AB_ROUNDS", "2"))
for r in range(rounds):
    for name, lib in variants:
        env = dict(os.environ, MHG_LIB=os.path.join(ROOT, lib), AB_ROOT=ROOT)
        res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = res.stdout.strip().splitlines()[-1] if res.returncode == 0 and res.stdout.strip() else res.stderr[-500:]
        print(f"round {r} {name:10s} {line}", flush=True)

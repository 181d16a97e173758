"""Same-process A/B of env-selected GEMM variants on short-K Schur views
(n=16384, 15360 x K x 15360, K = 1024 / 2048 / 15360): median of 5 interleaved
rounds of time_gemm(5) per variant.

  python profiles/ab_short.py name=ENV=VAL ...
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

n, q = 16384, int(os.environ.get("AB_Q", "65521"))
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
z = mh.encode(lay, 1024, 1024)
variants = [x.split("=", 1) for x in sys.argv[1:]] or [["default", "MHG_DUMMY=0"]]


class env_set:
    def __init__(self, spec):
        self.k, self.v = spec.split("=", 1)

    def __enter__(self):
        self.old = os.environ.get(self.k)
        os.environ[self.k] = self.v

    def __exit__(self, *a):
        if self.old is None:
            del os.environ[self.k]
        else:
            os.environ[self.k] = self.old


for K in (1024, 2048, 16384 - 1024):
    prob = mh.Problem(mh.Sub(A, z, 15360, 15360), mh.Sub(B, z, 15360, K), mh.Sub(C, z, K, 15360))
    plans = {}
    for name, env in variants:
        with env_set(env):
            plans[name] = mh.Plan(prob, mh.OP_SUB)
            plans[name].run()
    res = {name: [] for name, _ in variants}
    for r in range(int(os.environ.get("AB_ROUNDS", "5"))):
        for name, env in variants:
            # the GEMM parameters (and env hooks) are read at every time_gemm call
            with env_set(env):
                res[name].append(plans[name].time_gemm(5))
    print(f"K={K}: " + "  ".join(f"{nm} {statistics.median(v):.3f} ms" for nm, v in res.items()), flush=True)

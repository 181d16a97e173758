"""Diagnostic: replay test_random_misaligned_views' cases one by one (synchronising) to
find the first failing view shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1705_04807_b200 as mh
from oracle.binding import Oracle, OP_ADD, Views
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import _random_views, _views_from, _fill, _run_gpu
orc = Oracle()
for q in (2, 97, 257, 65521):
    op = OP_ADD
    rng = np.random.default_rng(q * 7 + op)
    for it in range(6):
        n = int(rng.choice([64, 128, 256]))
        t = int(rng.choice([x for x in (4, 8, 16, 32, 64) if x <= n]))
        r, k, c, corners = _random_views(rng, n)
        v = _views_from(orc, n, t, r, k, c, corners)
        out, lhs, rhs = _fill(orc, 1000 + it, n, q)
        print(f"q={q} it={it} n={n} t={t} r={r} k={k} c={c} corners={corners}", flush=True)
        got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, op)
        torch.cuda.synchronize()
        want = out.copy()
        orc.mm_dense(n, t, q, want, lhs, rhs, v, op=op)
        print("   ok" if np.array_equal(got, want) else "   MISMATCH", flush=True)

"""TU/TURBO-style update sweep on one Morton-hybrid parent (paper_1705_04807_b200.tu):
right-looking elimination updates A[k1:,k1:] -= A[k1:,k0:k1] A[k0:k1,k1:] with panel width
`block`, each step a graph-replayed aliased plan.  Reports GF(p) MAC/s over the sweep."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1705_04807_b200 as mh
from paper_1705_04807_b200.tu import schur_plans, schur_sweep
for n, block in [(16384, 1024), (16384, 2048), (16384, 1000), (32768, 2048)]:
    q = 65521
    f = torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda")
    M = mh.Matrix.wrap(mh.Layout(n, 64), mh.Modulus(q), f.data_ptr(), owner=f)
    plans = schur_plans(M, block)
    schur_sweep(M, block, plans=plans)  # warm-up / graph capture
    torch.cuda.synchronize()
    times = []
    for _ in range(7):  # the sweep's time varies run to run (clocks under the power cap)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        macs = schur_sweep(M, block, plans=plans)
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = sorted(times)[len(times) // 2]
    print(f"n={n} block={block} steps={len(plans)} median {ms:.2f} ms (min {min(times):.2f}, max "
          f"{max(times):.2f})  {macs / (ms * 1e-3):.3e} GF(p) MAC/s", flush=True)
    del plans, M, f; torch.cuda.empty_cache()

"""Row-major <-> Morton-hybrid conversion kernels (K1 k_rm_to_mh / k_mh_to_rm)
against the measured HBM copy bandwidth (cfg5 converts all three
operands).  Algorithmic bytes per call: 8 n^2 (4 read + 4 write).

  python profiles/conv_bench.py [n ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
q = 65521
# CONV=0/1/2: MHG_OPT_CONV_KERNEL (TMA / Morton-order LDG-STG / row-order)
modes = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("CONV=")] or [None]
for n in [int(a) for a in sys.argv[1:] if "=" not in a] or [16384, 32768]:
  for mode in modes:
    if mode is not None:
        mh.set_option(mh.OPT_CONV_KERNEL, int(mode))
    lay, mod = mh.Layout(n, 64), mh.Modulus(q)
    rm = torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda")
    back = torch.empty_like(rm)
    m = mh.Matrix(lay, mod)
    L = mh.lib()
    res = {}
    for name, fn in (("rm_to_mh", lambda: L.mhg_rowmajor_to_mh(m.handle, rm.data_ptr(), None)),
                     ("mh_to_rm", lambda: L.mhg_mh_to_rowmajor(m.handle, back.data_ptr(), None))):
        for _ in range(3):
            assert fn() == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 10
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        gbs = 8 * n * n / ms / 1e6
        res[name] = (ms, gbs)
    assert torch.equal(rm, back), "round trip mismatch"
    print(f"n={n} mode={mode}: " + "  ".join(f"{k} {ms:.3f} ms {g:.0f} GB/s ({g / peak:.2f} of {peak:.0f})"
                                 for k, (ms, g) in res.items()) +
          f"   3 operands rm->mh: {3 * res['rm_to_mh'][0]:.2f} ms", flush=True)
    del m, rm, back
    torch.cuda.empty_cache()

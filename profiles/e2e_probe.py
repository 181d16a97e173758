"""Where the e2e step goes: n=16384 uploads (16-bit wire) with and without a concurrent
1 GiB D2H per step, wall clock per step (10 steps).  python profiles/e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1705_04807_b200 as mh

n = 16384
lay, mod = mh.Layout(n, 64), mh.Modulus(65521)
mats = [mh.Matrix(lay, mod) for _ in range(3)]
hosts = [torch.randint(0, 65521, (n * n,), dtype=torch.int32).pin_memory() for _ in range(3)]
res = torch.empty(n * n, dtype=torch.int32).pin_memory()
dsrc = torch.empty(n * n, dtype=torch.int32, device="cuda")
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
lib = mh.lib()
for d2h in (False, True, False, True):
    for m, h in zip(mats, hosts):
        mh._check(lib.mhg_matrix_upload(m.handle, h.data_ptr(), s_up.cuda_stream))
    torch.cuda.synchronize()
    t = time.perf_counter()
    host_time = 0.0
    for _ in range(10):
        if d2h:
            with torch.cuda.stream(s_dn):
                res.copy_(dsrc, non_blocking=True)
        h0 = time.perf_counter()
        for m, h in zip(mats, hosts):
            mh._check(lib.mhg_matrix_upload(m.handle, h.data_ptr(), s_up.cuda_stream))
        host_time += time.perf_counter() - h0
        s_up.synchronize()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(f"3 uploads per step, concurrent 1 GiB D2H={d2h}: {dt * 1e3:.1f} ms/step "
          f"(host in upload calls {host_time / 10 * 1e3:.1f} ms)", flush=True)

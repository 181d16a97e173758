"""Upload of one n=16384 container (1 GiB of uint32 cells) from pinned host memory:
mhg_matrix_upload on the 16-bit wire vs a plain 4-byte cudaMemcpyAsync of the same
buffer.  Wall clock around enqueue + synchronize (the wire path's host narrowing is
part of the call).  Usage: python profiles/upload_wire.py [n] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1705_04807_b200 as mh

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
torch.cuda.set_device(0)
lay, mod = mh.Layout(n, 64), mh.Modulus(65521)
m = mh.Matrix(lay, mod)
host = torch.randint(0, 65521, (n * n,), dtype=torch.int32).pin_memory()
dev = torch.empty(n * n, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
lib = mh.lib()


def wire():
    mh._check(lib.mhg_matrix_upload(m.handle, host.data_ptr(), s.cuda_stream))


def plain():
    with torch.cuda.stream(s):
        dev.copy_(host, non_blocking=True)


for name, f in (("wire16", wire), ("plain32", plain)) * 2:
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{name}: {dt * 1e3:.2f} ms per 1 container ({n * n * 4 / dt / 1e9:.1f} GB/s of cells, "
          f"threads={os.environ.get('MHG_UPLOAD_THREADS', 'affinity')}, cpus={len(os.sched_getaffinity(0))})")
assert np.array_equal(m.cells(), host.numpy().view(np.uint32))
print("upload_bytes", m.upload_bytes)

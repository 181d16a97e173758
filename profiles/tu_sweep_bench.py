"""TU/TURBO-style update sweep on one Morton-hybrid parent (paper_1705_04807_b200.tu):
right-looking elimination updates A[k1:,k1:] -= A[k1:,k0:k1] A[k0:k1,k1:] with panel width
`block`, p = 65521, T' = 64.  Two timings per case, median of 7 (CUDA events):
  graph  -- the whole sweep captured into one CUDA graph (tu.SweepGraph): device-bound
  python -- one plan.run() per step from Python (host launch work between the steps)
plus the median SM clock (NVML) during the graph replays."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402
from paper_1705_04807_b200.tu import SweepGraph, schur_plans, schur_sweep  # noqa: E402

pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


def timed(fn, reps=7):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


cases = [(16384, 1024), (16384, 2048), (16384, 1000), (32768, 2048)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
for n, block in cases:
    q = 65521
    f = torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda")
    M = mh.Matrix.wrap(mh.Layout(n, 64), mh.Modulus(q), f.data_ptr(), owner=f)
    plans = schur_plans(M, block)
    schur_sweep(M, block, plans=plans)  # warm-up / per-plan graph capture
    sg = SweepGraph(M, block, plans=plans)
    sg.replay()
    torch.cuda.synchronize()
    clocks, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            time.sleep(0.002)
    th = threading.Thread(target=sample)
    th.start()
    ms_g = timed(sg.replay)
    stop.set()
    th.join()
    ms_p = timed(lambda: schur_sweep(M, block, plans=plans))
    mhz = statistics.median(clocks) if clocks else 0
    print(f"n={n} block={block} steps={len(plans)}  graph {ms_g:.2f} ms {sg.macs / (ms_g * 1e-3):.3e} GF(p) MAC/s "
          f"(SM {mhz:.0f} MHz)  python {ms_p:.2f} ms {sg.macs / (ms_p * 1e-3):.3e}", flush=True)
    del sg, plans, M, f
    torch.cuda.empty_cache()

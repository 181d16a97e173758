"""A/B harness for GEMM kernel variants under the power cap.

Interleaves variants in one process on the same operands, each for ~`secs`
seconds of back-to-back GEMM launches, sampling SM clock and board power with
NVML during each window.  Reports ms/launch, median MHz, mean W and
cycles/launch (ms x MHz) -- the clock-independent efficiency.

  python profiles/ab_gemm.py [n] [q] [rounds] [secs] variant=OPTION=VALUE ...
  e.g. python profiles/ab_gemm.py 16384 65521 3 2 pair=GEMM_KERNEL=2 1cta=GEMM_KERNEL=1
  (OPTION: an mhg option without the MHG_OPT_ prefix, include/mhg.h)
"""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_1705_04807_b200 as mh  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
variants = [a.split("=", 1) for a in sys.argv[1:] if "=" in a]
n = int(args[0]) if len(args) > 0 else 16384
q = int(args[1]) if len(args) > 1 else 65521
rounds = int(args[2]) if len(args) > 2 else 3
secs = float(args[3]) if len(args) > 3 else 2.0
if not variants:
    variants = [["pair", "GEMM_KERNEL=2"], ["1cta", "GEMM_KERNEL=1"]]


def opt(spec):
    k, v = spec.split("=", 1)
    return mh.options({getattr(mh, "OPT_" + k): int(v)})

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
fl = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda") for _ in range(3)]
A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
prob = mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n))
plans = {}
for name, spec in variants:
    with opt(spec):
        plans[name] = mh.Plan(prob, mh.OP_SUB)
        plans[name].run()
torch.cuda.synchronize()
macs = n ** 3


def sample(stop, clocks, watts):
    while not stop.is_set():
        clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        watts.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
        stop.wait(0.05)


res = {name: [] for name, _ in variants}
for r in range(rounds):
    for name, spec in variants:
      with opt(spec):
        pl = plans[name]
        pl.time_gemm(2)
        ms_one = pl.time_gemm(2)
        iters = max(3, int(secs * 1000 / max(ms_one, 0.01)))
        clocks, watts, stop = [], [], threading.Event()
        th = threading.Thread(target=sample, args=(stop, clocks, watts))
        th.start()
        ms = pl.time_gemm(iters)
        stop.set()
        th.join()
        mhz = statistics.median(clocks)
        res[name].append((ms, mhz, statistics.mean(watts)))
        print(f"round {r} {name:8s} {ms:8.3f} ms  {mhz:6.0f} MHz  {statistics.mean(watts):6.0f} W  "
              f"{ms * mhz / 1e3:8.1f} Mcyc  {macs / ms / 1e9:.3e} GF(p)MAC/s", flush=True)
for name, rs in res.items():
    ms = statistics.median(x[0] for x in rs)
    mhz = statistics.median(x[1] for x in rs)
    w = statistics.median(x[2] for x in rs)
    print(f"SUMMARY {name:8s} {ms:8.3f} ms  {mhz:6.0f} MHz  {w:6.0f} W  {ms * mhz / 1e3:8.1f} Mcyc")

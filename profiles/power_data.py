"""Power vs operand data: the same k_gemm on random residues, all zeros, and
residues with small signed digits, measuring clocks / watts / ms (NVML)."""
import os, statistics, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml, torch
import paper_1705_04807_b200 as mh
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
n, q = 16384, 65521
lay, mod = mh.Layout(n, 64), mh.Modulus(q)
def run(name, gen):
    fl = [gen() for _ in range(3)]
    A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl)
    pl = mh.Plan(mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n)), mh.OP_SUB)
    pl.run(); pl.time_gemm(3)
    clocks, watts, stop = [], [], threading.Event()
    def samp():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            watts.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000); stop.wait(0.05)
    th = threading.Thread(target=samp); th.start()
    ms = pl.time_gemm(200); stop.set(); th.join()
    print(f"{name:10s} {ms:7.3f} ms {statistics.median(clocks):6.0f} MHz {statistics.mean(watts):6.0f} W", flush=True)
    del pl, A, B, C, fl; torch.cuda.empty_cache()
run("random", lambda: torch.randint(0, q, (n*n,), dtype=torch.int32, device="cuda"))
run("zeros", lambda: torch.zeros(n*n, dtype=torch.int32, device="cuda"))
run("small", lambda: torch.randint(0, 16, (n*n,), dtype=torch.int32, device="cuda"))
run("random", lambda: torch.randint(0, q, (n*n,), dtype=torch.int32, device="cuda"))

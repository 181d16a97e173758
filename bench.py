#!/usr/bin/env python
"""Benchmark of the Morton-hybrid GF(p) MM hot path (BASELINE.json metric).

Default workload (N=1): n=16384, T'=64, p=65521, C -= A*B over full views --
the configuration BASELINE.json's metric is quoted on.  One step = one
planned multiply: pack(lhs) + pack(rhs) + tcgen05 GEMM with the fused mod-p
epilogue.  value = r*k*c GF(p) mult-adds per second (whole job).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload cfg2]

N > 1 runs under torchrun: C-stationary Morton-block partition, each rank
all-gathers its A row panel / B column panel (NCCL) and updates its block.
--impl reference times the reference's own CPU mm_oblivious (oracle/_ref) on
the host cores, on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P16, P31 = 65521, 2147483647
WORKLOADS = {
    # name: (n, t, q, op, view) ; view None = full n x n x n
    "ns16k": (16384, 64, P16, "sub", None),
    "cfg1": (512, 32, P16, "set", None),
    "cfg2": (4096, 64, P16, "sub", None),
    "cfg3": (8192, 64, P16, "sub", (96, 160, 6144, 2048, 5120)),
    "cfg4": (8192, 64, P31, "set", None),
    "cfg5": (32768, 64, P16, "sub", None),
}
DESCR = {
    "ns16k": "Morton-hybrid C -= A*B mod 65521, n=16384, T'=64 (north star)",
    "cfg1": "C = A*B mod 65521, n=512, T'=32",
    "cfg2": "C -= A*B mod 65521, n=4096, T'=64",
    "cfg3": "C(6144x5120) -= A(6144x2048)*B(2048x5120) mod 65521 in 8192^2 parents at (96,160), T'=64",
    "cfg4": "C = A*B mod 2^31-1, n=8192, T'=64",
    "cfg5": "C -= A*B mod 65521, n=32768, T'=64",
}
METRIC = "GF(p) mult-adds/s, Morton-hybrid C-=A·B mod p, n=16384; % of TC roofline"
UNIT = "GF(p) MAC/s"
DATA = ("synthetic: mh::Rng(0) -- std::mt19937_64, the reference's generator (bench.hpp:44-52) -- "
        "below(p) per cell in flat Morton order, out then lhs then rhs (gen_problem, bench.hpp:101-103); "
        "C zeroed for C = A*B workloads")


def config_of(workload):
    """The workload description both arms print (identical keys and values)."""
    n, t, q, op, view = WORKLOADS[workload]
    cfg = {"workload": workload, "description": DESCR[workload], "n": n, "t": t, "p": q, "op": op}
    if view is not None:
        cfg["view"] = {"row0": view[0], "col0": view[1], "rows": view[2], "inner": view[3], "cols": view[4]}
    gib = n * n * 4 / 2 ** 30
    size = "%.2f GiB" % gib if gib >= 1 else "%.0f MiB" % (gib * 1024)
    cfg["l2"] = ("no flush: operands 3 x %s %s 126 MB L2" % (size, ">>" if gib >= 0.25 else ">") if not fits_l2(n)
                 else "operands 3 x %.1f MiB fit in the 126 MB L2: L2 flushed before every timed step "
                      "(256 MiB memset), steps timed one by one" % (gib * 1024))
    return cfg


def fits_l2(n):
    """The three n x n uint32 containers fit in the B200's 126 MB L2 (cfg1): the timed loop
    then flushes L2 before every step."""
    return 3 * n * n * 4 <= (126 << 20)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def limbs_of(q):
    L = 1
    while q > 256 ** L:
        L += 1
    return L


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            float(d["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock + throttle reasons."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.1):
        self.samples, self.reasons = [], set()
        self.period, self.stop_evt = period, threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b and b != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop_evt.wait(self.period)

    def __enter__(self):
        if self.nv:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_evt.set()
            self.th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------- reference CPU leg
def reference_sample(n, t, q, threads, rows_per_thread=64, cols=512, view=None):
    """Time the reference's mm_oblivious (oracle/_ref, compiled from the
    reference's own headers) on a bounded sample of the workload: an output
    block of (64 x threads) rows x `cols` columns with the FULL inner length,
    split into one disjoint row strip per thread (multiply.hpp:25-29)."""
    from oracle.binding import REF_SO, Reference
    i0, j0, k0, inner = 0, 0, 0, n
    if view is not None:
        i0, j0, rr, inner, cc = view[0], view[1], view[2], view[3], view[4]
        k0 = view[1]
    if not os.path.exists(REF_SO):
        return None
    ref = Reference()
    h = ref.bench_new(n, t, q, 0)
    rows = min(rows_per_thread * threads, n - i0)
    cols = min(cols, n - j0)
    return ref, h, (i0, rows, j0, cols, k0, min(inner, n - k0))


def cpu_baseline_json(args, n, t, q, view, steps=1, warmup=0, one_core=True):
    threads = args.cpu_threads or os.cpu_count() or 1
    got = reference_sample(n, t, q, threads, view=view)
    if got is None:
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref/libmhref.so missing"}
    ref, h, (i0, rows, j0, cols, k0, inner) = got
    single = None
    try:
        for _ in range(warmup):
            ref.bench_run(h, i0, rows, j0, cols, k0, inner, threads)
        tot_ns, tot_macs = 0, 0
        for _ in range(steps):
            ns, macs = ref.bench_run(h, i0, rows, j0, cols, k0, inner, threads)
            tot_ns += ns
            tot_macs += macs
        if one_core:
            # the reference is single-threaded by contract (multiply.hpp:25-29): one call
            # on one core, a 64-row strip of the same sample
            ns1, macs1 = ref.bench_run(h, i0, min(64, rows), j0, cols, k0, inner, 1)
            single = {"value": macs1 / (ns1 * 1e-9), "unit": UNIT, "cores": 1,
                      "sample": f"one mh::mm_oblivious call on output rows [{i0},{i0 + min(64, rows)}) x "
                                f"cols [{j0},{j0 + cols}), inner {inner} ({macs1} MACs)"}
    finally:
        ref.bench_free(h)
    val = tot_macs / (tot_ns * 1e-9)
    return {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"mh::mm_oblivious (reference headers, -O3 -DNDEBUG) on output rows "
                      f"[{i0},{i0 + rows}) x cols [{j0},{j0 + cols}), inner {inner}, of the n={n} "
                      f"containers (mh::Rng(0) fill, as the GPU arm); {threads} disjoint row strips on "
                      f"{threads} std::threads; {steps} step(s) of {tot_macs // max(steps, 1)} MACs",
            "cpu_model": cpu_model(), "one_core": single,
            "ms_per_step": tot_ns / 1e6 / max(steps, 1)}


CPU_KEYS = ("value", "unit", "cores", "kind", "sample", "cpu_model", "one_core")


def run_reference(args, rank, world):
    n, t, q, op, view = WORKLOADS[args.workload]
    if rank != 0:
        return
    W = max(args.warmup, 0)
    cb = cpu_baseline_json(args, n, t, q, view, steps=args.steps, warmup=W)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": W, "ms_per_step": cb.get("ms_per_step"),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": DATA,
            "config": config_of(args.workload),
            "impl": "reference",
            "cpu_baseline": {k: cb.get(k) for k in CPU_KEYS},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg
def time_conversions(mh, torch, mats, n, q, hbm_gbs, reps=3):
    """Device row-major -> Morton of the three operands (K1, on-device residue check)
    and one Morton -> row-major, CUDA events; 8 n^2 algorithmic bytes per conversion."""
    lib = mh.lib()
    rm = torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda")
    back = torch.empty_like(rm)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for m in mats:  # warm-up
        assert lib.mhg_rowmajor_to_mh(m.handle, rm.data_ptr(), None) == 0
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        for m in mats:
            assert lib.mhg_rowmajor_to_mh(m.handle, rm.data_ptr(), None) == 0
    ev[1].record()
    ev[2].record()
    for _ in range(reps):
        assert lib.mhg_mh_to_rowmajor(mats[0].handle, back.data_ptr(), None) == 0
    ev[3].record()
    torch.cuda.synchronize()
    ok = bool(torch.equal(rm, back))
    to_mh = ev[0].elapsed_time(ev[1]) / (reps * len(mats))
    to_rm = ev[2].elapsed_time(ev[3]) / reps
    byts = 8 * n * n
    del rm, back
    torch.cuda.empty_cache()
    return {"rm_to_mh_ms": to_mh, "mh_to_rm_ms": to_rm, "three_operands_rm_to_mh_ms": 3 * to_mh,
            "rm_to_mh_gbs": byts / to_mh / 1e6, "mh_to_rm_gbs": byts / to_rm / 1e6,
            "frac_of_hbm": [byts / to_mh / 1e6 / hbm_gbs, byts / to_rm / 1e6 / hbm_gbs],
            "hbm_peak_gbs": hbm_gbs, "round_trip_exact": ok,
            "kernel": "k_conv_tma (2D tensor-map boxes <-> contiguous Morton runs, residue check in smem)"}


def e2e_pipelined(mh, torch, lay, mod, flats, set0, prob0, op, n, steps, macs, nsets=3):
    """End to end through the public C ABI with pinned HOST buffers: every step
    uploads its three inputs (mhg_matrix_upload), runs the plan, and downloads
    the result (mhg_matrix_download).  `nsets` container sets rotate so step i's
    result download (which waits for step i's compute) and the uploads of steps
    i+1 .. i+nsets-1 overlap: H2D, compute and D2H run on three streams ordered
    by events.  With 2 sets the uploads of step i+2 wait for step i's compute +
    download (~12 + ~23 ms at n = 16384); 3 sets keep the H2D stream busy."""
    hosts = []
    for f in flats:
        h = torch.empty(n * n, dtype=torch.int32, pin_memory=True)
        h.copy_(f)
        hosts.append(h)
    res = [torch.empty(n * n, dtype=torch.int32, pin_memory=True) for _ in range(nsets)]
    sets = [set0]
    for _ in range(nsets - 1):
        fl2 = [torch.empty_like(f) for f in flats]
        A2, B2, C2 = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in fl2)
        plan2 = mh.Plan(mh.Problem(mh.Sub(A2, prob0.a.origin, prob0.a.rows, prob0.a.cols),
                                   mh.Sub(B2, prob0.b.origin, prob0.b.rows, prob0.b.cols),
                                   mh.Sub(C2, prob0.c.origin, prob0.c.rows, prob0.c.cols)), op)
        sets.append((A2, B2, C2, plan2))
    s_up, s_cmp, s_dn = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_up = [torch.cuda.Event() for _ in range(nsets)]
    ev_cmp = [torch.cuda.Event() for _ in range(nsets)]
    ev_dn = [torch.cuda.Event() for _ in range(nsets)]
    lib = mh.lib()

    def one(i):
        k = i % nsets
        A_, B_, C_, pl = sets[k]
        if i >= nsets:  # container set k is free once its previous step was computed and read back
            s_up.wait_event(ev_cmp[k])
            s_up.wait_event(ev_dn[k])
        for h_, m_ in zip(hosts, (A_, B_, C_)):
            mh._check(lib.mhg_matrix_upload(m_.handle, h_.data_ptr(), s_up.cuda_stream))
        ev_up[k].record(s_up)
        s_cmp.wait_event(ev_up[k])
        pl.run(s_cmp)
        ev_cmp[k].record(s_cmp)
        s_dn.wait_event(ev_cmp[k])
        mh._check(lib.mhg_matrix_download(A_.handle, res[k].data_ptr(), s_dn.cuda_stream))
        ev_dn[k].record(s_dn)

    for i in range(nsets):  # warm-up of every set / graph
        one(i)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s_up)
    for i in range(steps):
        one(i)
    t1.record(s_dn)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    h2d = sum(m_.upload_bytes for m_ in sets[(steps - 1) % nsets][:3])  # PCIe bytes of the last step
    return {"value": macs / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": n * n * 4, "steps": steps, "ms_per_step": ms,
            "upload_wire": ("uint16" if h2d == 3 * n * n * 2 else "uint32" if h2d == 3 * n * n * 4 else "mixed"),
            "upload_adaptive": bool(mh.get_option(mh.OPT_UPLOAD_ADAPTIVE)), "container_sets": nsets,
            "path": "pinned host -> mhg_matrix_upload x3 (uint16 wire for q <= 2^16: host-threaded "
                    "narrowing into pinned staging, device widening) -> mhg_plan_run -> "
                    "mhg_matrix_download -> pinned host; %d container sets, H2D / compute / D2H "
                    "streams overlapped" % nsets}


def e2e_ranked(mh, torch, dist, mats, flats, out_f, step, stream, b, e, steps, macs, dev, barrier):
    """Multi-GPU end to end: each rank uploads its own 1/P slices from pinned
    host memory (mhg_matrix_upload_range: the 16-bit wire for q <= 2^16),
    exchanges panels, updates its C block, reads its slice back."""
    hosts = []
    for f in flats:
        h = torch.empty(e - b, dtype=torch.int32, pin_memory=True)
        h.copy_(f[b:e])
        hosts.append(h)
    res = torch.empty(e - b, dtype=torch.int32, pin_memory=True)
    torch.cuda.synchronize()
    barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(stream)
    for _ in range(steps):
        for h_, m_ in zip(hosts, mats):
            mh._check(mh.lib().mhg_matrix_upload_range(m_.handle, h_.data_ptr(), b, e - b,
                                                       stream.cuda_stream))
        step()  # segmented panel broadcasts overlapped with the per-segment GEMMs
        res.copy_(out_f[b:e], non_blocking=True)
    x1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t = torch.tensor([x0.elapsed_time(x1) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    h2d = sum(m_.upload_bytes for m_ in mats)
    return {"value": macs / (float(t[0]) * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": (e - b) * 4,
            "steps": steps, "ms_per_step": float(t[0]),
            "path": "per-rank pinned slices -> per segment: owner packs its A / B part "
                    "(mhg_plan_pack), packed limb planes exchanged (config.exchange) overlapped "
                    "with the segments' mhg_plan_gemm -> slice read-back"}


def seeded_containers(mh, torch, dev, n, q, b, e, zero_out=False, seed=0):
    """Three n x n device containers whose cells [b, e) hold mh::Rng(seed)'s draws in
    gen_problem's order (out, lhs, rhs; flat Morton order); the rest is zero."""
    import numpy as np
    g = mh.Rng(seed)
    chunk = 1 << 24
    host = torch.empty(chunk, dtype=torch.int32, pin_memory=True)
    hv = host.numpy().view(np.uint32)
    flats = []
    for which in range(3):
        f = torch.zeros(n * n, dtype=torch.int32, device=dev)
        pos = 0
        while pos < n * n:
            m = min(chunk, n * n - pos)
            g.below(q, m, out=hv[:m])
            lo, hi = max(pos, b), min(pos + m, e)
            if lo < hi and not (zero_out and which == 0):
                f[lo:hi].copy_(host[lo - pos:hi - pos], non_blocking=False)
            pos += m
        flats.append(f)
    torch.cuda.synchronize()
    return flats


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1705_04807_b200 as mh
    from paper_1705_04807_b200.dist import (PanelExchange, PeerPanels, PeerSetupError, exchange_bytes,
                                            rank_update, rank_update_packed, segment_plans, slice_range)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, t, q, opname, view = WORKLOADS[args.workload]
    op = {"add": mh.OP_ADD, "sub": mh.OP_SUB, "set": mh.OP_SET}[opname]
    L = limbs_of(q)
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    stream = torch.cuda.current_stream()
    shared_gpu = os.environ.get("MHG_BENCH_SHARED_GPU") == "1"

    # containers: full-size on every rank; each rank keeps its own 1/P Morton slice of
    # the reference's seed-0 stream (mh::Rng(0), gen_problem's fill order)
    b, e = slice_range(rank, world, n) if world > 1 else (0, n * n)
    flats = seeded_containers(mh, torch, dev, n, q, b, e, zero_out=(opname == "set"))
    out_f, lhs_f, rhs_f = flats
    A, B, Cm = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in flats)

    ex = PanelExchange(world, rank, n, t)
    if world > 1:
        blk = ex.block
        oi, oj, rr, kk, cc = blk.i0, blk.j0, blk.rows, n, blk.cols
        li, lj, ri, rj = blk.i0, 0, 0, blk.j0
        if view is not None:
            raise SystemExit("multi-GPU runs use full-view workloads")
    elif view is not None:
        oi, oj, rr, kk, cc = view
        li, lj, ri, rj = oi, oj, oi, oj
    else:
        oi = oj = li = lj = ri = rj = 0
        rr = kk = cc = n
    prob = mh.Problem(mh.Sub(A, mh.encode(lay, oi, oj), rr, cc),
                      mh.Sub(B, mh.encode(lay, li, lj), rr, kk),
                      mh.Sub(Cm, mh.encode(lay, ri, rj), kk, cc))
    macs_rank = rr * kk * cc
    macs_total = n ** 3 if world > 1 else macs_rank
    if world == 1:
        plans = [mh.Plan(prob, op)]
        segs = []
    else:
        # one plan per K segment: C[R_r, C_r] op= A[R_r, seg] B[seg, C_r]; the
        # segment's panels are broadcast while the previous segment computes
        segs = ex.segments()
        plans = segment_plans(mh, ex, A, B, Cm, op)
    plan = plans[0]
    info = plan.info()
    # N > 1 panel exchange: "p2p" (default) = packed limb planes pulled from the owners'
    # workspaces over CUDA IPC peer memory by the copy engines (no SMs taken from the
    # GEMM); "nccl" = the same bytes as NCCL broadcasts; "u32" = uint32 cells broadcast,
    # every rank packs its whole panels
    exchange = os.environ.get("MHG_EXCHANGE", "p2p") if world > 1 else "none"
    if exchange not in ("none", "p2p", "nccl", "u32"):
        raise SystemExit(f"MHG_EXCHANGE must be p2p, nccl or u32, got {exchange!r}")
    peer = None
    exchange_note = None
    if exchange == "p2p":
        # CPU-only barriers for the IPC event ordering (never wait for the GPU)
        host_group = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else None
        try:
            # ADD / SUB updates start with the segment of the rank's own row band (see PeerPanels)
            peer = PeerPanels(mh, ex, plans, host_group=host_group, rotate=(op != mh.OP_SET))
        except PeerSetupError as exc:  # collective: every rank falls back together
            exchange, exchange_note = "nccl", f"p2p setup failed, fell back to nccl: {exc}"[:300]
    if exchange in ("p2p", "nccl"):
        # packed exchange: one GEMM per segment + the packs of the parts this rank owns
        launches_per_step = sum(1 + (rank == sg.a_owner) + (rank == sg.b_owner) for sg in segs)
    else:
        launches_per_step = sum(pl.info()["launches"] for pl in plans)

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        if world == 1:
            plan.run(stream)
            return
        # packed limb planes on the wire (each owner packs its part; segment j+1's
        # pack + broadcasts are enqueued before segment j's GEMM); MHG_EXCHANGE=u32
        # exchanges the uint32 cells and packs every panel locally instead
        if exchange == "p2p":
            peer.update(stream)
        elif exchange == "u32":
            rank_update(ex, plans, lhs_f, rhs_f, stream)
        else:
            rank_update_packed(ex, plans, stream)

    gathered = [False]

    def verify_ranked():
        """N > 1: every rank checks its own C block on the device (Freivalds, mhg_verify).  That
        needs the whole A row panel and B column panel as residues, so the 1/P slices are
        gathered once into the (otherwise zero) full containers; the step itself still
        exchanges the packed planes as timed.  Collective; returns the minimum over ranks
        (None when memory is short: ranks sharing one GPU at n = 32768)."""
        torch.cuda.empty_cache()
        room = torch.tensor([float(torch.cuda.mem_get_info()[0] > 4 * n * n * (world if shared_gpu else 1)
                                   + (2 << 30))], dtype=torch.float64, device=dev)
        dist.all_reduce(room, op=dist.ReduceOp.MIN)  # one decision for every rank
        if room[0] < 0.5:
            return None
        if not gathered[0]:
            for f in (lhs_f, rhs_f):
                for r in range(world):
                    rb, re_ = slice_range(r, world, n)
                    dist.broadcast(f[rb:re_], src=r)
            gathered[0] = True
        old_f = out_f.clone()
        old = mh.Matrix.wrap(lay, mod, old_f.data_ptr(), owner=old_f)
        step()
        ok = mh.verify(prob, mh.Sub(old, prob.a.origin, prob.a.rows, prob.a.cols), op, rounds=2,
                       stream=stream)
        v = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MIN)
        del old, old_f
        torch.cuda.empty_cache()
        return bool(v[0] > 0.5)

    # The copy-engine exchange orders ranks through CUDA IPC events and peer mappings: check
    # one step of it on the device BEFORE timing; a wrong result (on any rank) sends every
    # rank to the NCCL packed exchange instead.
    if exchange == "p2p":
        step()
        # MHG_BENCH_FAIL_P2P_CHECK=1 (tests only) takes the fallback branch on a healthy exchange
        if verify_ranked() is False or os.environ.get("MHG_BENCH_FAIL_P2P_CHECK") == "1":
            torch.cuda.synchronize()
            barrier()
            peer.close()
            peer = None
            exchange, exchange_note = "nccl", "p2p failed the device verification, fell back to nccl"

    W = max(args.warmup, 3)
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the warm-up builds both graphs of every plan (plain and profiling, below): one profiled
    # step, then W plain ones (timed: they decide the loop layout)
    for pl in plans:
        pl.set_profiling(True)
    step()
    for pl in plans:
        pl.set_profiling(False)
        pl.gemm_time()
    w0.record(stream)
    for _ in range(W):
        step()
    w1.record(stream)
    torch.cuda.synchronize()
    barrier()
    warm_ms = w0.elapsed_time(w1) / W
    if world > 1:  # one decision for every rank (the loops below hold barriers)
        wt = torch.tensor([warm_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        warm_ms = float(wt[0])

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if fits_l2(n) else None

    def timed_loop(profiled):
        """K steps between device events (+ NVML clocks); profiled: every GEMM launch is
        bracketed by an event pair inside the plan's graph (its event-record nodes are
        re-pointed at the next ring pair per run, ~µs of host work per step)."""
        for pl in plans:
            pl.set_profiling(profiled)
            pl.gemm_time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pairs = []
        with ClockSampler(local_rank) as ck:
            torch.cuda.synchronize()
            barrier()
            e0.record(stream)
            for _ in range(args.steps):
                if flush is not None:
                    # operands that fit in L2: evict them (a write larger than L2) and time
                    # this step alone, so no step finds its inputs in L2
                    flush.zero_()
                    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    step()
                    b_.record(stream)
                    pairs.append((a, b_))
                else:
                    step()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
        g = 0.0  # per step: the rank's GEMM launches summed over its K segments
        for pl in plans:
            tot, cnt = pl.gemm_time()
            pl.set_profiling(False)
            g += tot / max(cnt, 1)
        if flush is not None:
            return sum(a.elapsed_time(b_) for a, b_ in pairs) / args.steps, ck, g
        return e0.elapsed_time(e1) / args.steps, ck, g

    # ---- timed region.  Steps of >= 1 ms: ONE loop, profiled (the per-GEMM event pairs cost
    # nothing there, and the GEMM times come from the timed steps themselves, same clocks).
    # Shorter steps (cfg1: ~15 us) would be host-bound by the profiling bookkeeping, so the
    # timed loop replays the plain graphs and a second, profiled loop gives the GEMM times.
    if warm_ms >= 1.0:
        ms_local, clk, gemm_ms = timed_loop(True)
        gemm_timing = {"loop": "the timed loop (GEMM launches bracketed by event-record graph nodes)"}
    else:
        ms_local, clk, _ = timed_loop(False)
        prof_ms, clk_prof, gemm_ms = timed_loop(True)
        gemm_timing = {"loop": "a second loop of the same steps, GEMM launches bracketed by event-record "
                               "graph nodes (host-bound at this step size, so not the timed loop)",
                       "ms_per_step": prof_ms, "clocks": clk_prof.summary()}
    t_ms = torch.tensor([ms_local, gemm_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms, gemm_ms_max = float(t_ms[0]), float(t_ms[1])
    value = macs_total / (ms * 1e-3)
    exchange_info = None
    if world > 1:
        # per rank: bytes received per step and the step time not covered by its GEMMs
        # (packs + exchange not hidden behind compute); max over ranks
        x = torch.tensor([float(exchange_bytes(ex, plans, exchange)), ms_local - gemm_ms], dtype=torch.float64,
                         device=dev)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        exchange_info = {"mode": exchange, "bytes_per_rank_step": int(x[0]),
                         "exposed_ms_per_step": float(x[1]),
                         "note": exchange_note}

    # ---- end to end through the public API with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        if world == 1:
            e2e = e2e_pipelined(mh, torch, lay, mod, flats, (A, B, Cm, plan), prob, op, n, e2e_steps,
                                macs_total, nsets=args.e2e_sets)
        else:
            e2e = e2e_ranked(mh, torch, dist, (A, B, Cm), flats, out_f, step, stream, b, e, e2e_steps,
                             macs_total, dev, barrier)
    # ---- one more step, checked on the device (Freivalds, mhg_verify) against a snapshot
    verified = None
    if world == 1:
        old_f = out_f.clone()
        old = mh.Matrix.wrap(lay, mod, old_f.data_ptr(), owner=old_f)
        step()
        verified = mh.verify(prob, mh.Sub(old, prob.a.origin, prob.a.rows, prob.a.cols), op, rounds=2,
                             stream=stream)
        del old, old_f
        torch.cuda.empty_cache()
    else:
        verified = verify_ranked()
    if peer is not None:
        torch.cuda.synchronize()
        barrier()
        peer.close()

    if rank != 0:
        return

    bf16_burst, bf16_sus, hbm, peak_src = load_peaks()
    int8_peak_tops = 2.0 * bf16_burst  # dense int8 = 2x dense bf16 on sm_100
    algo_ops = 2.0 * L * L * macs_rank  # int8 ops per GEMM launch (2 per limb MAC)
    achieved_tops = algo_ops / (gemm_ms_max * 1e-3) / 1e12
    traffic = tensor_pipe = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            rec = json.load(f).get(args.workload)
        if rec and world == 1:
            traffic = rec["dram_read"] + rec["dram_write"]
            tensor_pipe = rec.get("tensor_pipe_imma_active_pct")
    except Exception:
        traffic = None
    roof = {"bound": "tensor", "achieved": achieved_tops, "peak": int8_peak_tops,
            "unit": "TFLOP/s", "frac": achieved_tops / int8_peak_tops, "traffic": traffic,
            "traffic_source": "profiles/traffic.json (ncu --set full, bytes per launch)",
            "tensor_pipe_active_pct_ncu": tensor_pipe,
            "kernel": (f"k_gemm2<{L}> (tcgen05.mma.cta_group::2.kind::i8, CTA pair)"
                       if info.get("cta_group") == 2 else f"k_gemm<{L}> (tcgen05.mma.cta_group::1.kind::i8)")
                      + f", {info.get('digits')} digits",
            "peak_source": f"2 x {peak_src} bf16 burst {bf16_burst} TFLOP/s (MEASURED_PEAKS.json); "
                           f"int8 ops counted as 2*L^2*r*k*c, L={L}",
            "frac_of_spec_4500": achieved_tops / 4500.0,
            # 2 x the measured SUSTAINED bf16 rate (a seconds-long cuBLAS loop under the same 1 kW
            # cap): the denominator for long steps such as cfg5's ~100 ms x steps
            "frac_of_sustained": achieved_tops / (2.0 * bf16_sus),
            "gemm_ms": gemm_ms_max, "gemm_share_of_step": gemm_ms_max / ms, "gemm_timing": gemm_timing,
            "gf_macs_per_s_gemm_only": macs_rank / (gemm_ms_max * 1e-3)}
    # ---- row-major <-> Morton-hybrid conversion of all three operands,
    # timed separately after everything else (it overwrites the containers)
    conversion = None
    if world == 1:
        conversion = time_conversions(mh, torch, (A, B, Cm), n, q, hbm)
    cpu = None
    if not args.no_cpu_baseline:
        # rank 0 only, after every rank finished timing (the other ranks are idle)
        cb = cpu_baseline_json(args, n, t, q, view)
        cpu = {k: cb.get(k) for k in CPU_KEYS}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": W, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int8",
            "data": DATA,
            "config": config_of(args.workload),
            "verified": verified,
            "kernel_config": {"limbs": L,
                       "tiles": info["tiles"], "k_chunks": info["k_chunks"], "digits": info.get("digits"),
                       "partition": f"C-stationary Morton blocks over {world} GPU(s)"
                                    + ({"p2p": f", {len(plans)} K segments, packed limb planes "
                                               "pulled over CUDA IPC peer memory by the copy "
                                               "engines, overlapped with the per-segment GEMMs",
                                        "nccl": f", {len(plans)} K segments pipelined with NCCL "
                                                "broadcasts of packed limb planes",
                                        "u32": f", {len(plans)} K segments pipelined with NCCL "
                                               "broadcasts of uint32 cells"}.get(exchange, "")),
                       "exchange": exchange},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "conversion": conversion,
            "exchange": exchange_info,
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ns16k", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=30,
                    help="e2e steps (default = the device steps; the pipeline fill and drain are amortised over them)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-sets", type=int, default=3,
                    help="container sets rotated by the e2e pipeline (uploads run this many steps ahead)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # functional check of the N>1 path on ONE GPU (never a measurement): every rank on
    # cuda:0, collectives over gloo (host-staged).  No kernel waits on another rank.
    shared = os.environ.get("MHG_BENCH_SHARED_GPU") == "1"
    if shared:
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

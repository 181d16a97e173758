"""The multi-rank update path on real kernels: P = 2 and 4 ranks, each computing
its C-stationary Morton block through the segmented panel exchange and one
planned multiply per K segment (paper_1705_04807_b200.dist), must reproduce the
whole-container result of the oracle.  All ranks share cuda:0 and exchange over
gloo (host-staged): a functional check of the N>1 logic, never a measurement;
no kernel waits on another rank (B200_PROFILING.md, "kernels that wait on one
another")."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, t, q, op, outdir, mode="u32", steps=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_1705_04807_b200 as mh
    from paper_1705_04807_b200.dist import (PanelExchange, PeerPanels, rank_update,
                                            rank_update_packed, segment_plans, slice_range)

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(77)
        full = [rng.integers(0, q, n * n, dtype=np.uint32) for _ in range(3)]
        lo, hi = slice_range(rank, world, n)
        flats = []
        for f in full:  # every rank starts with only its own Morton slice
            d = torch.zeros(n * n, dtype=torch.int32, device="cuda")
            d[lo:hi] = torch.from_numpy(f[lo:hi].view(np.int32)).cuda()
            flats.append(d)
        lay, mod = mh.Layout(n, t), mh.Modulus(q)
        A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in flats)
        ex = PanelExchange(world, rank, n, t)
        plans = segment_plans(mh, ex, A, B, C, op)
        # ADD / SUB updates run the segments in each rank's rotated order (as bench.py does)
        peer = PeerPanels(mh, ex, plans, rotate=(op != mh.OP_SET)) if mode == "p2p" else None
        for _ in range(steps):
            if mode == "p2p":
                peer.update()
            elif mode == "packed":
                rank_update_packed(ex, plans)
            else:
                rank_update(ex, plans, flats[1], flats[2])
        torch.cuda.synchronize()
        dist.barrier()  # peers' pulls from this rank's workspaces are done
        if peer is not None:
            peer.close()
        np.save(os.path.join(outdir, f"slice{rank}.npy"), flats[0][lo:hi].cpu().numpy().view(np.uint32))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,op_name,mode,steps", [
    (2, "sub", "u32", 1), (4, "set", "u32", 1),
    (2, "sub", "packed", 1), (4, "sub", "packed", 1), (4, "set", "packed", 1),
    (2, "sub", "p2p", 1), (4, "sub", "p2p", 3), (4, "set", "p2p", 2), (8, "add", "p2p", 2)])
def test_multi_rank_update_matches_oracle(gpu, mh, oracle, tmp_path, world, op_name, mode, steps):
    """Every exchange mode: uint32 cells (rank_update), packed limb planes broadcast
    (rank_update_packed: owners pack, every rank runs only the GEMM) and packed
    planes pulled over CUDA IPC peer memory by the copy engines (PeerPanels);
    repeated steps check the cross-process event ordering (an owner's repack must
    wait for its pullers, a pull for the owner's pack)."""
    n, t, q = 256, 32, 65521
    from oracle.binding import OP_SET, OP_SUB, Views
    from oracle.binding import OP_ADD
    op = {"sub": mh.OP_SUB, "set": mh.OP_SET, "add": mh.OP_ADD}[op_name]
    oop = {"sub": OP_SUB, "set": OP_SET, "add": OP_ADD}[op_name]
    mp.spawn(_worker, args=(world, _free_port(), n, t, q, op, str(tmp_path), mode, steps),
             nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"slice{r}.npy") for r in range(world)])
    rng = np.random.default_rng(77)
    out, lhs, rhs = [rng.integers(0, q, n * n, dtype=np.uint32) for _ in range(3)]
    want = out.copy()
    for _ in range(steps):
        oracle.mm_dense(n, t, q, want, lhs, rhs, Views(0, 0, 0, n, n, n), op=oop)
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.slow
def test_bench_two_ranks_runs_end_to_end(gpu, mh, tmp_path):
    """bench.py --gpus 2 under torch.distributed.run (both ranks on cuda:0, gloo:
    MHG_BENCH_SHARED_GPU=1) prints one well-formed JSON line from rank 0."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MHG_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--workload", "cfg2", "--steps", "3", "--warmup", "3", "--e2e-steps", "2"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["verified"] is True and d["exchange"]["mode"] == "p2p"


def _fallback_worker(rank, world, port, outdir):
    """Rank 1 cannot map its peers' memory: every rank must raise PeerSetupError (the
    collective setup decision), after which the packed NCCL-style exchange runs."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_1705_04807_b200 as mh
    from paper_1705_04807_b200.dist import (PanelExchange, PeerPanels, PeerSetupError,
                                            rank_update_packed, segment_plans, slice_range)

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, t, q = 256, 32, 65521
        rng = np.random.default_rng(5)
        full = [rng.integers(0, q, n * n, dtype=np.uint32) for _ in range(3)]
        lo, hi = slice_range(rank, world, n)
        flats = []
        for f in full:
            d = torch.zeros(n * n, dtype=torch.int32, device="cuda")
            d[lo:hi] = torch.from_numpy(f[lo:hi].view(np.int32)).cuda()
            flats.append(d)
        lay, mod = mh.Layout(n, t), mh.Modulus(q)
        A, B, C = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in flats)
        ex = PanelExchange(world, rank, n, t)
        plans = segment_plans(mh, ex, A, B, C, mh.OP_SUB)
        if rank == 1:
            def refuse(handle):
                raise mh.DeviceError("simulated: no peer access")
            mh.ipc_open = refuse
        raised = False
        try:
            PeerPanels(mh, ex, plans)
        except PeerSetupError:
            raised = True
        rank_update_packed(ex, plans)
        torch.cuda.synchronize()
        dist.barrier()
        np.save(os.path.join(outdir, f"slice{rank}.npy"), flats[0][lo:hi].cpu().numpy().view(np.uint32))
        np.save(os.path.join(outdir, f"raised{rank}.npy"), np.array([raised]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_setup_failure_falls_back_collectively(gpu, mh, oracle, tmp_path):
    world = 4
    mp.spawn(_fallback_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all(bool(np.load(tmp_path / f"raised{r}.npy")[0]) for r in range(world))
    got = np.concatenate([np.load(tmp_path / f"slice{r}.npy") for r in range(world)])
    from oracle.binding import OP_SUB, Views
    n, t, q = 256, 32, 65521
    rng = np.random.default_rng(5)
    out, lhs, rhs = [rng.integers(0, q, n * n, dtype=np.uint32) for _ in range(3)]
    want = out.copy()
    oracle.mm_dense(n, t, q, want, lhs, rhs, Views(0, 0, 0, n, n, n), op=OP_SUB)
    assert np.array_equal(got, want)

"""Multi-GPU partitioning of C <- C +/- A*B by top-level Morton blocks of C.

One process per GPU (torch.distributed, NCCL on GPUs / gloo on CPU for tests).
With P = 2^b ranks, rank r owns the r-th contiguous 1/P slice of every
container's flat Morton-hybrid store.  Because the Z order visits quadrants
NW, NE, SW, SE at every scale (layout.hpp:42-48), that slice is a rectangle:
the bits of r, from the most significant, alternate (row half, column half)
choices of successive quadrant levels.  P=2: north/south halves; P=4: the four
quadrants; P=8: n/4 x n/2 blocks.

C is stationary: rank r updates only its own block C[R_r, C_r].  It needs the
A row panel A[R_r, :] and the B column panel B[:, C_r].  Those are the union of
the A slices of the ranks sharing its row band ("row group") and the B slices of
the ranks sharing its column band ("column group"), so the only exchange is an
all-gather inside each group -- no reduction, since K is never split.  This is
the reference's concurrency contract (disjoint output rectangles are
independent, multiply.hpp:25-29) applied across devices.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple


@dataclass(frozen=True)
class Block:
    rank: int
    i0: int
    j0: int
    rows: int
    cols: int
    row_band: int
    col_band: int


def _geom():
    """The partition geometry lives in libmhg.so (mhg_dist_*, include/mhg.h: pure host code,
    the same entry points a C++ host program would call)."""
    import paper_1705_04807_b200 as mh
    return mh


def _bits(P: int) -> int:
    if P < 1 or P & (P - 1):
        raise ValueError(f"rank count must be a power of two, got {P}")
    return P.bit_length() - 1


def morton_block(rank: int, P: int, n: int, t: int) -> Block:
    """Rectangle covered by the rank-th 1/P slice of an n x n Morton-hybrid store
    (mhg_dist_block)."""
    _bits(P)
    if not 0 <= rank < P:
        raise ValueError("rank out of range")
    if (n // t) ** 2 < P:
        raise ValueError("fewer tiles than ranks")
    b = _geom().dist_block(P, rank, n, t)
    return Block(rank, b.i0, b.j0, b.rows, b.cols, b.row_band, b.col_band)


def slice_range(rank: int, P: int, n: int) -> Tuple[int, int]:
    """Flat [begin, end) of the rank's slice of the Morton store (mhg_dist_slice)."""
    return _geom().dist_slice(P, rank, n)


def groups(P: int, n: int, t: int) -> Tuple[Dict[int, List[int]], Dict[int, List[int]]]:
    """row_band -> ranks sharing it, col_band -> ranks sharing it (ascending)."""
    rows: Dict[int, List[int]] = {}
    cols: Dict[int, List[int]] = {}
    for r in range(P):
        blk = morton_block(r, P, n, t)
        rows.setdefault(blk.row_band, []).append(r)
        cols.setdefault(blk.col_band, []).append(r)
    return rows, cols


@dataclass(frozen=True)
class Segment:
    """One K segment of rank r's update: C[R_r, C_r] op= A[R_r, k0:k1] B[k0:k1, C_r].

    The A part is a contiguous flat range of the row-group member `a_owner`'s
    Morton slice and the B part is the whole slice of column-group member
    `b_owner` (dyadic bands: the row bands refine the column bands, so K is cut
    at row-band boundaries)."""

    index: int
    k0: int
    k1: int
    a_owner: int
    a_range: Tuple[int, int]
    b_owner: int
    b_range: Tuple[int, int]


def segments(rank: int, P: int, n: int, t: int) -> List[Segment]:
    """The K segments of the rank's update (mhg_dist_segment)."""
    _bits(P)
    return [Segment(g.index, g.k0, g.k1, g.a_owner, (g.a_begin, g.a_end), g.b_owner,
                    (g.b_begin, g.b_end)) for g in _geom().dist_segments(P, rank, n, t)]


class PanelExchange:
    """Creates the row/column process groups once and all-gathers the panels
    each rank needs directly into its full-size containers (flat tensors)."""

    def __init__(self, P: int, rank: int, n: int, t: int):
        import torch.distributed as dist

        self.P, self.rank, self.n, self.t = P, rank, n, t
        self.block = morton_block(rank, P, n, t)
        rows, cols = groups(P, n, t)
        self.row_members = rows[self.block.row_band]
        self.col_members = cols[self.block.col_band]
        self.row_group = self.col_group = None
        if P > 1:
            # every rank must create every group, in the same order
            for band in sorted(rows):
                g = dist.new_group(rows[band])
                if band == self.block.row_band:
                    self.row_group = g
            for band in sorted(cols):
                g = dist.new_group(cols[band])
                if band == self.block.col_band:
                    self.col_group = g

    # -- pipelined form: one K segment at a time (overlaps the previous segment's GEMM)
    def segments(self) -> List[Segment]:
        return segments(self.rank, self.P, self.n, self.t)

    def exchange_segment(self, seg: Segment, lhs_flat, rhs_flat, async_op: bool = False):
        """Broadcast the segment's A part inside the row group and its B part
        inside the column group, in place in the full-size flat containers.
        Returns the pending work handles when async_op."""
        import torch.distributed as dist

        works = []
        if self.P == 1:
            return works
        for flat, owner, (b, e), members, group in (
                (lhs_flat, seg.a_owner, seg.a_range, self.row_members, self.row_group),
                (rhs_flat, seg.b_owner, seg.b_range, self.col_members, self.col_group)):
            if len(members) == 1:
                continue
            wk = dist.broadcast(flat[b:e], src=owner, group=group, async_op=async_op)
            if async_op:
                works.append(wk)
        return works

    def exchange(self, lhs_flat, rhs_flat):
        """lhs_flat / rhs_flat: the rank's full-size flat containers, holding its
        own slice; afterwards they hold the A row panel / B column panel."""
        import torch.distributed as dist

        if self.P == 1:
            return
        for flat, members, group in ((lhs_flat, self.row_members, self.row_group),
                                     (rhs_flat, self.col_members, self.col_group)):
            if len(members) == 1:
                continue
            parts = []
            for r in members:
                b, e = slice_range(r, self.P, self.n)
                parts.append(flat[b:e])
            mine = parts[members.index(self.rank)]
            dist.all_gather(parts, mine.clone(), group=group)


def segment_plans(mh, ex: PanelExchange, A, B, C, op: int):
    """One planned multiply per K segment of this rank's update
    C[R_r, C_r] op= A[R_r, seg] * B[seg, C_r] (A = out, B = lhs, C = rhs in the
    reference's Problem order).  A SET update overwrites only with the first
    segment; the rest accumulate."""
    return [mh.Plan.for_segment(A, B, C, op, ex.P, ex.rank, j) for j in range(len(ex.segments()))]


def rank_update(ex: PanelExchange, plans, lhs_flat, rhs_flat, stream=None):
    """This rank's whole update: segment j+1's panel broadcasts are enqueued before
    segment j's multiply so the exchange overlaps compute (NCCL on GPUs)."""
    segs = ex.segments()
    pending = ex.exchange_segment(segs[0], lhs_flat, rhs_flat, async_op=True)
    for j, pl in enumerate(plans):
        for wk in pending:
            wk.wait()
        pending = (ex.exchange_segment(segs[j + 1], lhs_flat, rhs_flat, async_op=True)
                   if j + 1 < len(segs) else [])
        pl.run(stream)


def rank_update_packed(ex: PanelExchange, plans, stream=None):
    """This rank's update with PACKED panels on the wire (2-byte limb
    planes for p < 2^16 instead of uint32 cells): for every K segment, the owner
    of the A part packs it into its segment plan's workspace and broadcasts the
    packed bytes inside the row group (all members hold plans of the same lhs
    geometry), the B part likewise inside the column group; every rank then runs
    the segment's GEMM on the received packs.  Each rank packs only its own data.
    Segment j+1's pack + broadcasts are enqueued before segment j's GEMM."""
    import torch.distributed as dist

    segs = ex.segments()

    def issue(j):
        sg, pl, works = segs[j], plans[j], []
        for which, owner, members, group in ((0, sg.a_owner, ex.row_members, ex.row_group),
                                             (1, sg.b_owner, ex.col_members, ex.col_group)):
            if ex.rank == owner:
                pl.pack(which, stream)
            if len(members) > 1:
                works.append(dist.broadcast(pl.pack_buffer(which), src=owner, group=group,
                                            async_op=True))
        return works

    pending = issue(0)
    for j, pl in enumerate(plans):
        for wk in pending:
            wk.wait()
        pending = issue(j + 1) if j + 1 < len(plans) else []
        pl.gemm(stream)


def pull_lists(ex: PanelExchange):
    """Which packed parts this rank pulls, and which ranks pull from it.

    Returns (pulls, pullers): pulls[j] = [(which, owner)] for segment j (which =
    0: the A part, 1: the B part), pullers = the ranks that pull any part from
    this one.  An owner packs segment j's part into ITS OWN segment-j plan, so
    the pull reads the owner's plan j: every member of a row group sees the same
    A owner for segment j, and every member of a column group the same B owner
    (tests/test_dist_gloo.py checks this for P up to 16)."""
    pulls, pullers = [], set()
    for sg in ex.segments():
        row = []
        for which, owner, members in ((0, sg.a_owner, ex.row_members),
                                      (1, sg.b_owner, ex.col_members)):
            if owner == ex.rank:
                pullers.update(m for m in members if m != ex.rank)
            else:
                row.append((which, owner))
        pulls.append(row)
    return pulls, pullers


class PeerSetupError(RuntimeError):
    """Peer-memory setup failed on some rank (every rank raises it)."""


def exchange_bytes(ex: PanelExchange, plans, mode: str) -> int:
    """Bytes this rank receives per step: packed planes of the parts it does not own
    (p2p, nccl) or the uint32 slices of its row / column group (u32)."""
    if ex.P == 1:
        return 0
    total = 0
    for sg, pl in zip(ex.segments(), plans):
        for which, owner, members, rng in ((0, sg.a_owner, ex.row_members, sg.a_range),
                                           (1, sg.b_owner, ex.col_members, sg.b_range)):
            if owner == ex.rank or len(members) == 1:
                continue
            total += pl.pack_region(which)[1] if mode in ("p2p", "nccl") else 4 * (rng[1] - rng[0])
    return total


class PeerPanels:
    """Copy-engine exchange of the PACKED panels over NVLink peer memory.

    Same data movement as rank_update_packed (each owner packs its part of every
    segment once; the members of its row / column group need those bytes), but
    the bytes move as cudaMemcpyAsync pulls from the owner's workspace, mapped
    once through CUDA IPC, instead of NCCL broadcasts.  Copies run on the copy
    engines, so the persistent GEMM keeps all SMs (an NCCL kernel would hold
    some of them while it runs beside the GEMM), and every segment's pulls are
    enqueued at once, one copy stream per owner, each GEMM waiting only for its
    own segment.

    Ordering is by CUDA IPC events, so no stream ever blocks the host:
      pack_done[j]  recorded by an owner after packing its parts of segment j;
                    pullers' copy streams wait on it before pulling segment j;
      copy_done     recorded by a puller after its last pull; an owner's next
                    pack waits on it before overwriting the workspace.
    Each cross-process wait is enqueued after a host barrier that follows the
    matching record (the IPC event contract), on `host_group` (gloo: a CPU-only
    barrier that never waits for the GPU).  No kernel waits on another rank's
    kernel: the waits are stream-level dependencies, so the path is exercised
    safely with all ranks on one GPU (tests/test_dist_gpu.py).

    The owner's packs run on a high-priority side stream, one event per segment, so
    its own segment-j GEMM waits only for pack j (and segment j's pulls), not for the
    packs of later segments.

    Setup is collective: if mapping a peer's memory fails on any rank (no peer access
    between the devices, IPC unsupported), every rank raises PeerSetupError and the
    caller can fall back to the NCCL exchange (rank_update_packed)."""

    def __init__(self, mh, ex: PanelExchange, plans, host_group=None, device=None, rotate=False):
        import torch
        import torch.distributed as dist

        self.mh, self.ex, self.plans = mh, ex, plans
        self.bases = {}
        self.group = host_group
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.segs = ex.segments()
        # Processing order of the K segments.  rotate: start with the segment of the rank's own
        # row band -- its B part is the rank's own slice (no pull) and its A part is what the
        # row-group owner packs first, so the first GEMM waits for one small pull instead of
        # two; B parts of the later segments belong to ranks that packed them first.  Sums
        # commute, but a SET update must run segment 0 (the overwriting plan) first: callers
        # rotate only ADD / SUB updates.
        S = len(self.segs)
        first = ex.block.row_band % S if rotate and S else 0
        self.order = [(first + d) % S for d in range(S)]
        rank, P = ex.rank, ex.P
        ev = lambda: torch.cuda.Event(enable_timing=False, blocking=False, interprocess=True)
        self.pack_done = [ev() for _ in self.segs]
        self.copy_done = ev()
        exports = {}
        mine = {"error": None}
        try:  # an export that fails here is reported collectively below, like a failed mapping
            for j, (sg, pl) in enumerate(zip(self.segs, plans)):
                for which, owner in ((0, sg.a_owner), (1, sg.b_owner)):
                    ptr, nb = pl.pack_region(which)
                    if owner == rank and nb:
                        h, off = mh.ipc_export(ptr)
                        exports[(j, which)] = (h, off, nb)
            mine.update({"exports": exports, "pack_done": [e.ipc_handle() for e in self.pack_done],
                         "copy_done": self.copy_done.ipc_handle()})
        except Exception as exc:  # noqa: BLE001
            mine["error"] = f"rank {rank}: export failed: {exc}"
        infos = [None] * P
        dist.all_gather_object(infos, mine, group=host_group)
        failed = [i["error"] for i in infos if i["error"]]
        if failed:
            raise PeerSetupError("; ".join(failed))
        # pulls[j] = [(owner, dst, src, bytes)]; one mapping per owner allocation
        self.pulls = [[] for _ in self.segs]
        owners = set()
        lists, pullers = pull_lists(ex)
        error = None
        try:
            for j, pl in enumerate(plans):
                for which, owner in lists[j]:
                    dst, nb = pl.pack_region(which)
                    if not nb:
                        continue
                    h, off, onb = infos[owner]["exports"][(j, which)]
                    if onb != nb:
                        raise RuntimeError(f"segment {j}: packed sizes differ ({onb} vs {nb})")
                    if h not in self.bases:
                        self.bases[h] = mh.ipc_open(h)
                    self.pulls[j].append((owner, dst, self.bases[h] + off, nb))
                    owners.add(owner)
            self.peer_pack_done = {o: [torch.cuda.Event.from_ipc_handle(self.device, hnd)
                                       for hnd in infos[o]["pack_done"]] for o in sorted(owners)}
            self.peer_copy_done = [torch.cuda.Event.from_ipc_handle(self.device, infos[p]["copy_done"])
                                   for p in sorted(pullers)]
        except Exception as exc:  # noqa: BLE001 -- reported collectively below
            error = f"rank {rank}: {exc}"
        errors = [None] * P
        dist.all_gather_object(errors, error, group=host_group)
        failed = [e for e in errors if e]
        if failed:
            self.close()
            raise PeerSetupError("; ".join(failed))
        self.pull_bytes = sum(nb for pulls in self.pulls for (_, _, _, nb) in pulls)
        self.pack_stream = torch.cuda.Stream(device=self.device, priority=-1)
        self.copy_streams = {o: torch.cuda.Stream(device=self.device) for o in sorted(owners)}
        self.join = torch.cuda.Stream(device=self.device)
        # per (segment, owner): "this owner's pulls of the segment have landed"
        self.landed = [{o: torch.cuda.Event() for o in {pull[0] for pull in pulls}}
                       for pulls in self.pulls]
        self.dst_free = torch.cuda.Event()
        self.steps = 0

    def _barrier(self):
        import torch.distributed as dist
        dist.barrier(group=self.group)

    def close(self):
        for base in self.bases.values():
            self.mh.ipc_close(base)
        self.bases = {}

    def update(self, stream=None):
        """One whole update of this rank's C block (all K segments)."""
        import torch

        stream = torch.cuda.current_stream(self.device) if stream is None else stream
        rank = self.ex.rank
        ps = self.pack_stream
        self._barrier()  # every puller recorded copy_done of the previous step
        # packs overwrite workspaces this rank's previous GEMMs and its pullers read
        ps.wait_stream(stream)
        if self.steps:
            for e in self.peer_copy_done:
                ps.wait_event(e)
        for j in self.order:
            sg, pl = self.segs[j], self.plans[j]
            if sg.a_owner == rank:
                pl.pack(0, ps)
            if sg.b_owner == rank:
                pl.pack(1, ps)
            self.pack_done[j].record(ps)
        # this rank's pulls overwrite workspaces its previous GEMMs read
        self.dst_free.record(stream)
        self._barrier()  # every owner recorded pack_done of this step
        for cs in self.copy_streams.values():
            cs.wait_event(self.dst_free)
        for j in self.order:
            pulls = self.pulls[j]
            used = []
            for owner, dst, src, nb in pulls:
                cs = self.copy_streams[owner]
                if owner not in used:
                    cs.wait_event(self.peer_pack_done[owner][j])
                    used.append(owner)
                self.mh.copy_async(dst, src, nb, cs)
            for owner in used:
                ev = self.landed[j][owner]
                ev.record(self.copy_streams[owner])
                stream.wait_event(ev)
                self.join.wait_event(ev)
            stream.wait_event(self.pack_done[j])  # this rank's own parts of segment j
            self.plans[j].gemm(stream)
        self.copy_done.record(self.join)
        self.steps += 1


def rank_update_p2p(peer: PeerPanels, stream=None):
    """This rank's update with packed panels pulled over peer memory (PeerPanels)."""
    peer.update(stream)

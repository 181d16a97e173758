"""Multi-rank host logic of the C-stationary Morton-block partition, on CPU
with the gloo backend (world sizes 2 and 4): every rank ends up holding exactly
the A row panel and B column panel its C block needs, and the blocks tile C."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1705_04807_b200.dist import PanelExchange, groups, morton_block, slice_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_blocks_tile_the_matrix_and_match_morton_slices(oracle):
    n, t = 64, 4
    for P in (1, 2, 4, 8, 16):
        cover = np.zeros((n, n), np.int32)
        for r in range(P):
            b = morton_block(r, P, n, t)
            cover[b.i0:b.i0 + b.rows, b.j0:b.j0 + b.cols] += 1
            lo, hi = slice_range(r, P, n)
            # the block is exactly the set of cells stored in the rank's flat slice
            zs = {oracle.encode(n, t, i, j) for i in range(b.i0, b.i0 + b.rows)
                  for j in range(b.j0, b.j0 + b.cols)}
            assert zs == set(range(lo, hi))
        assert (cover == 1).all()
    rows, cols = groups(8, n, t)
    assert all(len(v) == 2 for v in rows.values()) and all(len(v) == 4 for v in cols.values())
    with pytest.raises(ValueError):
        morton_block(0, 3, n, t)


def test_segments_are_exact_flat_ranges(oracle):
    """Every K segment's A part / B part is exactly one contiguous flat range of
    its owner's Morton slice (what the broadcasts move), and the segments tile K."""
    from paper_1705_04807_b200.dist import segments
    n, t = 32, 4
    for P in (1, 2, 4, 8, 16):
        for r in range(P):
            blk = morton_block(r, P, n, t)
            segs = segments(r, P, n, t)
            assert [s.k0 for s in segs] == sorted(s.k0 for s in segs)
            assert segs[0].k0 == 0 and segs[-1].k1 == n
            assert all(a.k1 == b.k0 for a, b in zip(segs, segs[1:]))
            for sg in segs:
                za = {oracle.encode(n, t, i, j) for i in range(blk.i0, blk.i0 + blk.rows)
                      for j in range(sg.k0, sg.k1)}
                zb = {oracle.encode(n, t, i, j) for i in range(sg.k0, sg.k1)
                      for j in range(blk.j0, blk.j0 + blk.cols)}
                assert za == set(range(*sg.a_range)) and zb == set(range(*sg.b_range))



# ---- the C ABI's partition geometry (mhg_dist_*, include/mhg.h) against an independent
# restatement of the same rules in Python
def _py_block(rank, P, n):
    b = P.bit_length() - 1
    row_bits, col_bits = (b + 1) // 2, b // 2
    rb = cb = 0
    for k in range(b):  # from the most significant bit of rank
        bit = (rank >> (b - 1 - k)) & 1
        if k % 2 == 0:
            rb = (rb << 1) | bit
        else:
            cb = (cb << 1) | bit
    rows, cols = n >> row_bits, n >> col_bits
    return rb * rows, cb * cols, rows, cols, rb, cb


def _py_segments(rank, P, n):
    b = P.bit_length() - 1
    row_bits, col_bits = (b + 1) // 2, b // 2
    h, w = n >> row_bits, n >> col_bits
    per = n * n // P
    owners = {_py_block(r, P, n)[4:]: r for r in range(P)}
    _, _, _, _, rband, cband = _py_block(rank, P, n)
    out = []
    for i in range(1 << row_bits):
        k0 = i * h
        a_owner = owners[(rband, k0 // w)]
        half = per // (w // h)
        part = (k0 % w) // h
        b_owner = owners[(i, cband)]
        out.append((i, k0, k0 + h, a_owner, a_owner * per + part * half, a_owner * per + (part + 1) * half,
                    b_owner, b_owner * per, (b_owner + 1) * per))
    return out


def test_c_abi_partition_geometry(mh):
    for n, t in ((64, 4), (96, 3), (512, 32), (16384, 64), (32768, 64)):
        for P in (1, 2, 4, 8, 16, 32, 64):
            if (n // t) ** 2 < P:
                continue
            for r in range(P):
                b = mh.dist_block(P, r, n, t)
                assert (b.i0, b.j0, b.rows, b.cols, b.row_band, b.col_band) == _py_block(r, P, n)
                assert b.rank == r
                assert mh.dist_slice(P, r, n) == (r * (n * n // P), (r + 1) * (n * n // P))
                got = [(g.index, g.k0, g.k1, g.a_owner, g.a_begin, g.a_end, g.b_owner, g.b_begin, g.b_end)
                       for g in mh.dist_segments(P, r, n, t)]
                assert got == _py_segments(r, P, n)
    with pytest.raises(mh.InvalidArgument):
        mh.dist_block(3, 0, 64, 4)          # not a power of two
    with pytest.raises(mh.InvalidArgument):
        mh.dist_block(0, 0, 64, 4)
    with pytest.raises(mh.OutOfRange):
        mh.dist_block(4, 4, 64, 4)          # rank out of range
    with pytest.raises(mh.InvalidArgument):
        mh.dist_block(32, 0, 16, 4)         # 16 tiles, 32 ranks
    with pytest.raises(mh.InvalidArgument):
        mh.dist_block(2, 0, 12, 4)          # not a layout
    with pytest.raises(mh.OutOfRange):
        mh.dist_slice(4, 7, 64)
    with pytest.raises(mh.InvalidArgument):
        mh.dist_segments(6, 0, 64, 4)


def test_rotated_segment_order_starts_on_the_ranks_own_b_part(mh):
    """PeerPanels(rotate=True) starts each rank on the K segment of its own row band: the
    segment whose B part is the rank's own slice (nothing to pull for it) -- and every
    row-group member starts on the same segment, so the A-part owner packs it first."""
    from paper_1705_04807_b200.dist import segments
    n, t = 256, 32
    for P in (2, 4, 8, 16):
        for r in range(P):
            blk = morton_block(r, P, n, t)
            segs = segments(r, P, n, t)
            first = segs[blk.row_band % len(segs)]
            assert first.b_owner == r and first.b_range == slice_range(r, P, n)
            # the A part of that segment comes from the rank's own row group
            assert morton_block(first.a_owner, P, n, t).row_band == blk.row_band


def _seg_worker(rank, world, port, n, t, q, use_async):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full_a = torch.arange(n * n, dtype=torch.int32) % q + 1
        full_b = (torch.arange(n * n, dtype=torch.int32) * 7) % q + 1
        lo, hi = slice_range(rank, world, n)
        a = torch.zeros(n * n, dtype=torch.int32)
        b = torch.zeros(n * n, dtype=torch.int32)
        a[lo:hi], b[lo:hi] = full_a[lo:hi], full_b[lo:hi]
        ex = PanelExchange(world, rank, n, t)
        for sg in ex.segments():
            for wk in ex.exchange_segment(sg, a, b, async_op=use_async):
                wk.wait()
            # after segment sg arrives, its A and B parts are present
            assert torch.equal(a[sg.a_range[0]:sg.a_range[1]], full_a[sg.a_range[0]:sg.a_range[1]])
            assert torch.equal(b[sg.b_range[0]:sg.b_range[1]], full_b[sg.b_range[0]:sg.b_range[1]])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,use_async", [(2, False), (4, True)])
def test_segmented_exchange_gloo(world, use_async):
    mp.spawn(_seg_worker, args=(world, _free_port(), 32, 4, 97, use_async), nprocs=world, join=True)


def _worker(rank, world, port, n, t, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full_a = torch.arange(n * n, dtype=torch.int32) % q + 1
        full_b = (torch.arange(n * n, dtype=torch.int32) * 7) % q + 1
        lo, hi = slice_range(rank, world, n)
        a = torch.zeros(n * n, dtype=torch.int32)
        b = torch.zeros(n * n, dtype=torch.int32)
        a[lo:hi] = full_a[lo:hi]
        b[lo:hi] = full_b[lo:hi]
        ex = PanelExchange(world, rank, n, t)
        ex.exchange(a, b)
        blk = ex.block
        from oracle.binding import Oracle
        orc = Oracle()
        # A row panel rows [i0, i0+rows) x all columns; B column panel all rows x [j0, j0+cols)
        need_a = [orc.encode(n, t, i, j) for i in range(blk.i0, blk.i0 + blk.rows) for j in range(n)]
        need_b = [orc.encode(n, t, i, j) for i in range(n) for j in range(blk.j0, blk.j0 + blk.cols)]
        assert torch.equal(a[need_a], full_a[need_a])
        assert torch.equal(b[need_b], full_b[need_b])
        # nothing outside the needed panels was received (traffic = panels only)
        mask = torch.zeros(n * n, dtype=torch.bool)
        mask[need_a] = True
        mask[lo:hi] = True
        assert (a[~mask] == 0).all()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_panel_exchange_gloo(world):
    mp.spawn(_worker, args=(world, _free_port(), 32, 4, 97), nprocs=world, join=True)


def test_peer_pull_lists_read_the_owners_own_segment_plan():
    """PeerPanels pulls segment j's packed part from the owner's segment-j plan:
    that plan must pack exactly the same part (same K range, same flat range, same
    panel height / width), and the puller / owner relations must be symmetric."""
    from types import SimpleNamespace

    from paper_1705_04807_b200.dist import pull_lists, segments

    n, t = 256, 8
    for P in (1, 2, 4, 8, 16):
        rows, cols = groups(P, n, t)
        exs = []
        for r in range(P):
            b = morton_block(r, P, n, t)
            exs.append(SimpleNamespace(rank=r, P=P, block=b, row_members=rows[b.row_band],
                                       col_members=cols[b.col_band],
                                       segments=lambda r=r: segments(r, P, n, t)))
        lists = [pull_lists(ex) for ex in exs]
        pulled_from = {r: set() for r in range(P)}
        for r, ex in enumerate(exs):
            pulls, _ = lists[r]
            mine = ex.segments()
            assert len(pulls) == len(mine)
            for j, row in enumerate(pulls):
                got = {w for w, _ in row}
                # every part is either this rank's own or pulled, never both
                assert got == {w for w, o in ((0, mine[j].a_owner), (1, mine[j].b_owner)) if o != r}
                for which, owner in row:
                    pulled_from[owner].add(r)
                    theirs = exs[owner].segments()[j]
                    assert (theirs.k0, theirs.k1) == (mine[j].k0, mine[j].k1)
                    if which == 0:
                        assert theirs.a_owner == owner and theirs.a_range == mine[j].a_range
                        assert exs[owner].block.rows == ex.block.rows
                    else:
                        assert theirs.b_owner == owner and theirs.b_range == mine[j].b_range
                        assert exs[owner].block.cols == ex.block.cols
        for r in range(P):
            assert lists[r][1] == pulled_from[r]
        if P == 1:
            assert lists[0] == ([[]], set())

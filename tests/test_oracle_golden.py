"""Pins the CPU oracle (oracle/mh_oracle.c) against the reference's golden
vectors and against the reference library itself (oracle/_ref).  CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.binding import OP_ADD, OP_SET, OP_SUB, Views

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f) if name.endswith(".json") else f.read()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


# ------------------------------------------------------------------ codec
def test_encode_pinned_values(oracle):
    """layout_test.cpp:30-41"""
    assert oracle.encode(8, 4, 0, 0) == 0
    assert oracle.encode(8, 4, 2, 5) == 25
    assert oracle.encode(8, 4, 5, 6) == 54
    assert oracle.extract(8, 4, 25) == (2, 5)
    assert oracle.extract(8, 4, 47) == (7, 3)


def _z_walk(bi, bj, side, out):
    """Independent recursive NW, NE, SW, SE tile walk (oracles.hpp:18-42)."""
    if side == 1:
        out.append((bi, bj))
        return
    h = side // 2
    _z_walk(bi, bj, h, out)
    _z_walk(bi, bj + h, h, out)
    _z_walk(bi + h, bj, h, out)
    _z_walk(bi + h, bj + h, h, out)


@pytest.mark.parametrize("n,t", [(4, 1), (8, 4), (16, 4), (16, 2), (24, 3), (32, 8)])
def test_encode_follows_quadrant_walk(oracle, n, t):
    """layout_test.cpp:43-56"""
    blocks = []
    _z_walk(0, 0, n // t, blocks)
    z = 0
    for (bi, bj) in blocks:
        for li in range(t):
            for lj in range(t):
                i, j = bi * t + li, bj * t + lj
                assert oracle.encode(n, t, i, j) == z
                assert oracle.extract(n, t, z) == (i, j)
                z += 1


def test_rowmajor_roundtrip(oracle):
    """matrix.hpp:44-67 / layout_test.cpp:108-145"""
    rng = np.random.default_rng(0)
    for n, t in [(8, 4), (24, 3), (64, 8)]:
        g = rng.integers(0, 1000, (n, n), dtype=np.uint32)
        cells = oracle.rowmajor_to_mh(n, t, g)
        assert np.array_equal(oracle.mh_to_rowmajor(n, t, cells), g)


# ------------------------------------------------------------------ field
def test_field_kats(oracle):
    """field_test.cpp:65-71 (q = 2^31 - 1)"""
    q = 2147483647
    assert oracle.lib.orc_mul(q - 1, q - 2, q) == 2
    assert oracle.lib.orc_add(q - 1, q - 2, q) == q - 3
    assert oracle.lib.orc_is_prime(65521) and not oracle.lib.orc_is_prime(65535)


# -------------------------------------------------------------- generator
def test_first_draw_seed0(oracle):
    """bench_test.cpp:56-72: descriptor triple and container hash."""
    g = _load("first_draw_seed0_n64_t8_q2.json")
    out, lhs, rhs, aligned, v = oracle.gen_problem(oracle.rng(0), 64, 8, 2)
    assert (v.out_origin, v.rows, v.cols) == (1, 64, 39) == (g["out_origin"], g["rows"], g["cols"])
    assert (v.lhs_origin, v.inner) == (322, 3)
    assert v.rhs_origin == 2855
    assert not aligned
    h = 0
    for x in out.tolist():
        h = (h * 31 + x) & (2 ** 64 - 1)
    assert h == 4715125990397575263 == g["out_hash31"]


def test_twenty_trial_golden_counts(oracle):
    """bench_test.cpp:74-115: the oblivious base-case counts and MACs of the
    seed-0 20-trial batch, from the restated draws + recursion."""
    rows = _load("bench_trials_seed0_n64_t8_q2.csv").strip().splitlines()
    assert rows[0] == "trial,sigmaA,rA,cA,sigmaB,rB,cB,sigmaC,rC,cC,calls_default,calls_obl,macs"
    g = oracle.rng(0)
    for ln in rows[1:]:
        f = [int(x) for x in ln.split(",")]
        out, lhs, rhs, _, v = oracle.gen_problem(g, 64, 8, 2)
        assert [v.out_origin, v.rows, v.cols, v.lhs_origin, v.rows, v.inner, v.rhs_origin,
                v.inner, v.cols] == f[1:10]
        ctr = oracle.mm_oblivious(64, 8, 2, out, lhs, rhs, v)
        assert ctr.base_case_calls == f[11]
        assert ctr.scalar_macs == f[12]
        assert ctr.encode_calls == 0 and ctr.max_consecutive_jump <= 8


def test_frozen_seed0_grid(oracle):
    """multiply_test.cpp:134-163 through the dense oracle and the recursion."""
    gd = _load("frozen_seed0_gf2.json")
    frozen = [[1, 0, 0, 0], [1, 0, 1, 1], [0, 1, 0, 1], [1, 0, 1, 0]]
    assert gd["frozen_view"] == frozen
    g = oracle.rng(0)
    grids = [np.array([g.next() % 2 for _ in range(64)], np.uint32).reshape(8, 8) for _ in range(3)]
    assert [gr.tolist() for gr in grids] == gd["grids_rowmajor"]
    cells = [oracle.rowmajor_to_mh(8, 4, gr) for gr in grids]
    v = Views(oracle.encode(8, 4, 1, 2), oracle.encode(8, 4, 3, 1), oracle.encode(8, 4, 2, 4), 4, 4, 4)
    for method in ("dense", "oblivious"):
        a = cells[0].copy()
        if method == "dense":
            oracle.mm_dense(8, 4, 2, a, cells[1], cells[2], v)
        else:
            oracle.mm_oblivious(8, 4, 2, a, cells[1], cells[2], v)
        assert oracle.mh_to_rowmajor(8, 4, a).tolist() == gd["result_rowmajor"]


def test_golden_cases_oracle(oracle):
    """Reference-generated cases: oracle output hash and Counters match."""
    for c in _load("cases.json"):
        n, t, q = c["n"], c["t"], c["q"]
        g = oracle.rng(c["seed"])
        for _ in range(c["draw"]):
            oracle.gen_problem(g, n, t, q)
        out, lhs, rhs, _, v = oracle.gen_problem(g, n, t, q)
        assert [v.out_origin, v.lhs_origin, v.rhs_origin, v.rows, v.inner, v.cols] == c["views"]
        a = out.copy()
        oracle.mm_dense(n, t, q, a, lhs, rhs, v, op=c["op"], threads=2)
        assert sha(a) == c["out_sha256"], c
        if c["op"] == OP_ADD:
            b = out.copy()
            assert list(oracle.mm_oblivious(n, t, q, b, lhs, rhs, v).as_tuple()) == c["counters"]
            assert sha(b) == c["out_sha256"]


# ---------------------------------------------- oracle vs the reference itself
@pytest.mark.parametrize("n,t,q,seed,count", [(64, 8, 2, 101, 60), (64, 8, 97, 102, 60),
                                              (256, 32, 2, 103, 8)])
def test_oracle_equals_reference(oracle, reference, n, t, q, seed, count):
    """acceptance_main.cpp:177-217 configurations: restated recursion and dense
    oracle agree cell for cell with the reference's mm_oblivious, Counters too."""
    g = oracle.rng(seed)
    for _ in range(count):
        out, lhs, rhs, _, v = oracle.gen_problem(g, n, t, q)
        a, b, c = out.copy(), out.copy(), out.copy()
        ref = reference.mm_oblivious(n, t, q, a, lhs, rhs, v)
        mine = oracle.mm_oblivious(n, t, q, b, lhs, rhs, v)
        oracle.mm_dense(n, t, q, c, lhs, rhs, v, threads=2)
        assert np.array_equal(a, b) and np.array_equal(a, c)
        assert ref.as_tuple() == mine.as_tuple()
        assert ref.scalar_macs == v.rows * v.inner * v.cols


def test_reference_csv_golden(reference, tmp_path):
    """The reference's own run_trials CSV (time columns stripped) equals the
    committed golden (which equals bench_test.cpp:528-549)."""
    p = str(tmp_path / "t.csv")
    reference.run_trials_csv(64, 8, 2, 0, 20, 2, p)
    got = "\n".join(",".join(l.split(",")[:-2]) for l in open(p).read().splitlines()) + "\n"
    assert got == _load("bench_trials_seed0_n64_t8_q2.csv")


def test_sub_and_set_semantics(oracle, reference):
    """C -= A*B == C += (-A)*B and C = A*B on the view only, vs the reference."""
    g = oracle.rng(5)
    for _ in range(10):
        out, lhs, rhs, _, v = oracle.gen_problem(g, 32, 4, 97)
        for op in (OP_SUB, OP_SET):
            a, b = out.copy(), out.copy()
            reference.mm_oblivious(32, 4, 97, a, lhs, rhs, v, op=op)
            oracle.mm_dense(32, 4, 97, b, lhs, rhs, v, op=op, threads=1)
            assert np.array_equal(a, b)


# ------------------------------------------------------- size-free checkers
def test_freivalds_and_blocks(oracle):
    n, t, q = 128, 16, 65521
    g = oracle.rng(9)
    out, lhs, rhs = (oracle.fill_below(g, n * n, q) for _ in range(3))
    v = Views(oracle.encode(n, t, 5, 7), oracle.encode(n, t, 5, 3), oracle.encode(n, t, 9, 7),
              100, 90, 110)
    for op in (OP_ADD, OP_SUB, OP_SET):
        new = out.copy()
        oracle.mm_dense(n, t, q, new, lhs, rhs, v, op=op)
        assert oracle.freivalds(n, t, q, out, lhs, rhs, new, v, op=op, rounds=3)
        blk = oracle.mm_dense_block(n, t, q, out, lhs, rhs, v, 10, 20, 30, 40, op=op)
        for a in range(20):
            for b in range(40):
                assert blk[a, b] == new[oracle.encode(n, t, 5 + 10 + a, 7 + 30 + b)]
        bad = new.copy()
        z = oracle.encode(n, t, 50, 50)
        bad[z] = (bad[z] + 1) % q
        assert not oracle.freivalds(n, t, q, out, lhs, rhs, bad, v, op=op, rounds=1)

"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``    -- oracle/liboracle.so, the plain-C restatement of the reference path
                   (oracle/mh_oracle.c, citations inside).
* ``Reference`` -- oracle/_ref/libmhref.so, the reference library itself compiled
                   in place from /root/reference by oracle/Makefile.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmhref.so")

U32P = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
U64 = C.c_uint64


class Counters(C.Structure):
    """multiply.hpp:39-45"""

    _fields_ = [
        ("base_case_calls", U64),
        ("scalar_macs", U64),
        ("encode_calls", U64),
        ("recursive_calls", U64),
        ("max_consecutive_jump", U64),
    ]

    def as_tuple(self):
        return (self.base_case_calls, self.scalar_macs, self.encode_calls,
                self.recursive_calls, self.max_consecutive_jump)


class _Problem(C.Structure):
    _fields_ = [
        ("n", U64), ("t", U64), ("q", C.c_uint32),
        ("out", C.c_void_p), ("lhs", C.c_void_p), ("rhs", C.c_void_p),
        ("out_origin", U64), ("lhs_origin", U64), ("rhs_origin", U64),
        ("rows", U64), ("inner", U64), ("cols", U64),
    ]


@dataclass
class Views:
    """A problem's three views: out (rows x cols) op= lhs (rows x inner) * rhs."""

    out_origin: int
    lhs_origin: int
    rhs_origin: int
    rows: int
    inner: int
    cols: int


OP_ADD, OP_SUB, OP_SET = 0, 1, 2


def _build_hint(path):
    return f"{path} missing: run `make -C oracle` (or __graft_entry__.build())"


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(_build_hint(path))
        L = C.CDLL(path)
        self.lib = L
        L.orc_rng_new.restype = C.c_void_p
        L.orc_rng_new.argtypes = [U64]
        L.orc_rng_free.argtypes = [C.c_void_p]
        L.orc_rng_next.restype = U64
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_rng_below.restype = U64
        L.orc_rng_below.argtypes = [C.c_void_p, U64]
        L.orc_fill_below.argtypes = [C.c_void_p, U32P, U64, C.c_uint32]
        L.orc_is_prime.argtypes = [C.c_uint32]
        L.orc_add.restype = C.c_uint32
        L.orc_add.argtypes = [C.c_uint32] * 3
        L.orc_mul.restype = C.c_uint32
        L.orc_mul.argtypes = [C.c_uint32] * 3
        L.orc_layout_check.argtypes = [U64, U64]
        for f in ("orc_encode",):
            getattr(L, f).restype = U64
            getattr(L, f).argtypes = [U64] * 4
        for f in ("orc_extract_i", "orc_extract_j"):
            getattr(L, f).restype = U64
            getattr(L, f).argtypes = [U64] * 3
        L.orc_dilate.restype = U64
        L.orc_dilate.argtypes = [U64]
        L.orc_gen_problem.argtypes = [C.c_void_p, U64, U64, C.c_uint32, U32P, U32P, U32P,
                                      np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")]
        L.orc_mm_oblivious.argtypes = [C.POINTER(_Problem), C.POINTER(Counters)]
        L.orc_mm_dense.argtypes = [C.POINTER(_Problem), C.c_int, C.c_int]
        L.orc_mm_dense_block.argtypes = [C.POINTER(_Problem), C.c_int, U64, U64, U64, U64, U32P, C.c_int]
        L.orc_freivalds.argtypes = [C.POINTER(_Problem), U32P, C.c_int, C.c_int, U64, C.c_int]
        L.orc_rowmajor_to_mh.argtypes = [U64, U64, U32P, U32P]
        L.orc_mh_to_rowmajor.argtypes = [U64, U64, U32P, U32P]

    # -- generator
    def rng(self, seed: int):
        return _Rng(self.lib, seed)

    def fill_below(self, rng, count: int, q: int) -> np.ndarray:
        a = np.empty(count, dtype=np.uint32)
        self.lib.orc_fill_below(rng.h, a, count, q)
        return a

    def gen_problem(self, rng, n, t, q):
        out = np.empty(n * n, np.uint32)
        lhs = np.empty(n * n, np.uint32)
        rhs = np.empty(n * n, np.uint32)
        desc = np.zeros(10, np.uint64)
        st = self.lib.orc_gen_problem(rng.h, n, t, q, out, lhs, rhs, desc)
        if st:
            raise ValueError(f"gen_problem status {st}")
        d = [int(x) for x in desc]
        return out, lhs, rhs, bool(d[0]), Views(d[1], d[4], d[7], d[2], d[6], d[3])

    # -- codec
    def encode(self, n, t, i, j):
        return int(self.lib.orc_encode(n, t, i, j))

    def extract(self, n, t, z):
        return int(self.lib.orc_extract_i(n, t, z)), int(self.lib.orc_extract_j(n, t, z))

    def rowmajor_to_mh(self, n, t, rows: np.ndarray) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.uint32).reshape(-1)
        out = np.empty(n * n, np.uint32)
        if self.lib.orc_rowmajor_to_mh(n, t, rows, out):
            raise ValueError("bad layout")
        return out

    def mh_to_rowmajor(self, n, t, cells: np.ndarray) -> np.ndarray:
        out = np.empty(n * n, np.uint32)
        if self.lib.orc_mh_to_rowmajor(n, t, np.ascontiguousarray(cells, dtype=np.uint32), out):
            raise ValueError("bad layout")
        return out.reshape(n, n)

    # -- multiply
    @staticmethod
    def _problem(n, t, q, out, lhs, rhs, v: Views) -> _Problem:
        for a in (out, lhs, rhs):
            assert a.dtype == np.uint32 and a.flags.c_contiguous and a.size == n * n
        return _Problem(n, t, q, out.ctypes.data, lhs.ctypes.data, rhs.ctypes.data,
                        v.out_origin, v.lhs_origin, v.rhs_origin, v.rows, v.inner, v.cols)

    def mm_oblivious(self, n, t, q, out, lhs, rhs, v: Views) -> Counters:
        p = self._problem(n, t, q, out, lhs, rhs, v)
        ctr = Counters()
        st = self.lib.orc_mm_oblivious(C.byref(p), C.byref(ctr))
        if st:
            raise _status_error(st)
        return ctr

    def mm_dense(self, n, t, q, out, lhs, rhs, v: Views, op=OP_ADD, threads=None):
        p = self._problem(n, t, q, out, lhs, rhs, v)
        st = self.lib.orc_mm_dense(C.byref(p), op, threads or os.cpu_count() or 1)
        if st:
            raise _status_error(st)

    def mm_dense_block(self, n, t, q, out, lhs, rhs, v: Views, r0, nr, c0, nc, op=OP_ADD,
                       threads=None) -> np.ndarray:
        p = self._problem(n, t, q, out, lhs, rhs, v)
        dst = np.empty(nr * nc, np.uint32)
        st = self.lib.orc_mm_dense_block(C.byref(p), op, r0, nr, c0, nc, dst,
                                         threads or os.cpu_count() or 1)
        if st:
            raise _status_error(st)
        return dst.reshape(nr, nc)

    def freivalds(self, n, t, q, old_out, lhs, rhs, new_out, v: Views, op=OP_ADD, rounds=2,
                  seed=1234, threads=None) -> bool:
        p = self._problem(n, t, q, old_out, lhs, rhs, v)
        r = self.lib.orc_freivalds(C.byref(p), np.ascontiguousarray(new_out), op, rounds, seed,
                                   threads or os.cpu_count() or 1)
        if r < 0:
            raise _status_error(-r)
        return r == 1


class _Rng:
    def __init__(self, lib, seed):
        self.lib = lib
        self.h = lib.orc_rng_new(seed)

    def next(self):
        return int(self.lib.orc_rng_next(self.h))

    def below(self, k):
        return int(self.lib.orc_rng_below(self.h, k))

    def __del__(self):
        try:
            self.lib.orc_rng_free(self.h)
        except Exception:
            pass


def _status_error(st):
    return {1: ValueError, 2: IndexError, 3: RuntimeError}.get(st, OSError)(f"status {st}")


class Reference:
    """The reference library itself (oracle/_ref/libmhref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(_build_hint(path))
        L = C.CDLL(path)
        self.lib = L
        L.ref_encode.argtypes = [U64, U64, U64, U64, C.POINTER(U64)]
        L.ref_extract.argtypes = [U64, U64, U64, C.POINTER(U64), C.POINTER(U64)]
        L.ref_mm.argtypes = [C.c_int, U64, U64, C.c_uint32, U32P, U64, U64, U64, U32P, U64, U64,
                             U32P, U64, C.c_int, C.POINTER(Counters)]
        L.ref_counters_mixed.argtypes = [C.c_int] + [U64] * 12 + [C.POINTER(Counters)]
        L.ref_save_matrix.argtypes = [U64, U64, C.c_uint32, U64, C.c_char_p]
        L.ref_gen_problem.argtypes = [U64, U64, C.c_uint32, U64, C.c_uint32, U32P, U32P, U32P,
                                      np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")]
        L.ref_run_trials_csv.argtypes = [U64, U64, C.c_uint32, U64, C.c_uint32, C.c_int, C.c_char_p]
        L.ref_bench_new.restype = C.c_void_p
        L.ref_bench_new.argtypes = [U64, U64, C.c_uint32, U64]
        L.ref_bench_free.argtypes = [C.c_void_p]
        L.ref_bench_run.restype = C.c_longlong
        L.ref_bench_run.argtypes = [C.c_void_p, U64, U64, U64, U64, U64, U64, C.c_int, C.POINTER(U64)]

    def encode(self, n, t, i, j):
        z = U64()
        st = self.lib.ref_encode(n, t, i, j, C.byref(z))
        if st:
            raise _status_error(st)
        return z.value

    def mm(self, kind, n, t, q, out, lhs, rhs, v: Views, op=OP_ADD) -> Counters:
        ctr = Counters()
        st = self.lib.ref_mm(kind, n, t, q, out, v.out_origin, v.rows, v.cols, lhs, v.lhs_origin,
                             v.inner, rhs, v.rhs_origin, op, C.byref(ctr))
        if st:
            raise _status_error(st)
        return ctr

    def mm_oblivious(self, *a, **k):
        return self.mm(2, *a, **k)

    def save_matrix(self, n, t, q, seed, path):
        """The reference's save_matrix_file on an mh::Rng(seed)-filled container."""
        st = self.lib.ref_save_matrix(n, t, q, seed, path.encode())
        if st:
            raise _status_error(st)

    def counters_mixed(self, kind, geo_out, geo_lhs, geo_rhs, rows, inner, cols) -> Counters:
        """Counters of mm_naive (kind 0) / mm_default (1); geo_* = (n, t, origin) per container."""
        ctr = Counters()
        st = self.lib.ref_counters_mixed(kind, *geo_out, *geo_lhs, *geo_rhs, rows, inner, cols,
                                         C.byref(ctr))
        if st:
            raise _status_error(st)
        return ctr

    def gen_problem(self, n, t, q, seed, skip=0):
        out = np.empty(n * n, np.uint32)
        lhs = np.empty(n * n, np.uint32)
        rhs = np.empty(n * n, np.uint32)
        desc = np.zeros(10, np.uint64)
        st = self.lib.ref_gen_problem(n, t, q, seed, skip, out, lhs, rhs, desc)
        if st:
            raise _status_error(st)
        d = [int(x) for x in desc]
        return out, lhs, rhs, bool(d[0]), Views(d[1], d[4], d[7], d[2], d[6], d[3])

    def run_trials_csv(self, n, t, q, seed, trials, algo, path):
        st = self.lib.ref_run_trials_csv(n, t, q, seed, trials, algo, path.encode())
        if st:
            raise _status_error(st)

    # -- CPU baseline timing
    def bench_new(self, n, t, q, seed=0):
        h = self.lib.ref_bench_new(n, t, q, seed)
        if not h:
            raise MemoryError("ref_bench_new failed")
        return h

    def bench_run(self, h, i0, rows, j0, cols, k0, inner, threads):
        macs = U64()
        ns = self.lib.ref_bench_run(h, i0, rows, j0, cols, k0, inner, threads, C.byref(macs))
        if ns < 0:
            raise RuntimeError("ref_bench_run failed")
        return ns, macs.value

    def bench_free(self, h):
        self.lib.ref_bench_free(h)

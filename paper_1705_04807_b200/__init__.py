"""B200-native Morton-hybrid GF(p) matrix multiplication (C <- C +/- A*B mod p).

Python mirror of the reference's header API (arxiv/paper_1705_04807,
proj/include/mh) over the C ABI of libmhg.so (include/mhg.h).  Names and
argument meanings follow the reference:

    Layout(n, t), encode / extract_i / extract_j        layout.hpp:42-99
    Modulus(q), Fp arithmetic                            field.hpp:23-55
    Matrix(layout, modulus), from_row_major, to_row_major  matrix.hpp:13-67
    Sub(mat, origin, rows, cols)                         submatrix.hpp:13-18
    Problem(a=out, b=lhs, c=rhs), Counters               multiply.hpp:39-53
    mm_oblivious(problem) -> Counters                    multiply.hpp:297-308

Error behaviour mirrors the reference's exception classes:
    std::invalid_argument -> InvalidArgument (a ValueError)
    std::out_of_range     -> OutOfRange      (an IndexError)
    std::logic_error      -> LogicError      (a RuntimeError)

All compute runs in the sm_100a kernels of libmhg.so.  There is no CPU
fallback: importing works anywhere (codec/validation are host code), but any
device call fails loudly with DeviceError when the library or an sm_100 GPU is
missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = [
    "InvalidArgument", "OutOfRange", "LogicError", "DeviceError", "Unsupported",
    "Layout", "Modulus", "Matrix", "Sub", "Problem", "Counters", "Plan",
    "encode", "extract_i", "extract_j", "from_row_major", "to_row_major",
    "mm_oblivious", "mm_naive", "mm_default", "mm", "counters_oblivious", "counters_layout",
    "counters_geometry", "limb_params", "lib", "LIB_PATH", "KERNEL_NAIVE", "KERNEL_DEFAULT",
    "verify", "Rng",
    "Sweep", "DistBlock", "DistSegment", "dist_block", "dist_slice", "dist_segments",
    "OP_ADD", "OP_SUB", "OP_SET", "set_option", "get_option", "options",
    "OPT_DIGITS", "OPT_GEMM_KERNEL", "OPT_MIN_FOLD_LEVEL", "OPT_MAX_KCHUNK", "OPT_UPLOAD_WIRE",
    "OPT_CONV_KERNEL", "OPT_GEMM_STATS", "OPT_UPLOAD_THREADS", "OPT_UPLOAD_ADAPTIVE",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# MHG_LIB: an alternative build of the same library (kernel A/B diagnostics only)
LIB_PATH = os.environ.get("MHG_LIB") or os.path.join(HERE, "libmhg.so")
OP_ADD, OP_SUB, OP_SET = 0, 1, 2
# mhg_option keys (include/mhg.h)
(OPT_DIGITS, OPT_GEMM_KERNEL, OPT_MIN_FOLD_LEVEL, OPT_MAX_KCHUNK, OPT_UPLOAD_WIRE, OPT_CONV_KERNEL,
 OPT_GEMM_STATS, OPT_UPLOAD_THREADS, OPT_UPLOAD_ADAPTIVE) = range(1, 10)


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class LogicError(RuntimeError):
    """std::logic_error"""


class DeviceError(RuntimeError):
    """CUDA failure, missing library or no sm_100 device (no fallback)."""


class Unsupported(RuntimeError):
    """Valid for the reference, not supported by this build."""


_ERR = {1: InvalidArgument, 2: OutOfRange, 3: LogicError, 4: DeviceError, 5: Unsupported}


class _View(C.Structure):
    _fields_ = [("mat", C.c_void_p), ("origin", C.c_uint64), ("rows", C.c_uint64),
                ("cols", C.c_uint64)]


class IpcHandle(C.Structure):
    """mhg_ipc_handle (include/mhg.h): a cudaIpcMemHandle_t as 64 opaque bytes."""

    _fields_ = [("bytes", C.c_ubyte * 64)]


class DistBlock(C.Structure):
    """mhg_dist_block_t: a rank's block of every container (include/mhg.h)."""

    _fields_ = [("rank", C.c_uint32), ("i0", C.c_uint64), ("j0", C.c_uint64), ("rows", C.c_uint64),
                ("cols", C.c_uint64), ("row_band", C.c_uint32), ("col_band", C.c_uint32)]


class DistSegment(C.Structure):
    """mhg_dist_segment_t: one K segment of a rank's update and the owners of its parts."""

    _fields_ = [("index", C.c_uint32), ("k0", C.c_uint64), ("k1", C.c_uint64),
                ("a_owner", C.c_uint32), ("a_begin", C.c_uint64), ("a_end", C.c_uint64),
                ("b_owner", C.c_uint32), ("b_begin", C.c_uint64), ("b_end", C.c_uint64)]


class Counters(C.Structure):
    """multiply.hpp:39-45"""

    _fields_ = [("base_case_calls", C.c_uint64), ("scalar_macs", C.c_uint64),
                ("encode_calls", C.c_uint64), ("recursive_calls", C.c_uint64),
                ("max_consecutive_jump", C.c_uint64)]

    def as_tuple(self):
        return (self.base_case_calls, self.scalar_macs, self.encode_calls,
                self.recursive_calls, self.max_consecutive_jump)

    def __repr__(self):
        return "Counters(%s)" % ", ".join(f"{n}={getattr(self, n)}" for n, _ in self._fields_)


_lib = None


def lib():
    """Load libmhg.so (built in-tree by __graft_entry__.build() / make)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    u64, u32, vp = C.c_uint64, C.c_uint32, C.c_void_p
    P = C.POINTER
    sigs = {
        "mhg_last_error": ([], C.c_char_p),
        "mhg_version": ([], C.c_char_p),
        "mhg_device_check": ([], C.c_int),
        "mhg_set_option": ([C.c_int, C.c_int64], C.c_int),
        "mhg_get_option": ([C.c_int, P(C.c_int64)], C.c_int),
        "mhg_layout_check": ([u64, u64], C.c_int),
        "mhg_modulus_check": ([u32], C.c_int),
        "mhg_encode": ([u64, u64, u64, u64, P(u64)], C.c_int),
        "mhg_extract": ([u64, u64, u64, P(u64), P(u64)], C.c_int),
        "mhg_matrix_create": ([u64, u64, u32, P(vp)], C.c_int),
        "mhg_matrix_wrap": ([u64, u64, u32, vp, P(vp)], C.c_int),
        "mhg_matrix_destroy": ([vp], C.c_int),
        "mhg_matrix_info": ([vp, P(u64), P(u64), P(u32), P(vp)], C.c_int),
        "mhg_matrix_upload": ([vp, vp, vp], C.c_int),
        "mhg_matrix_upload_bytes": ([vp, P(u64)], C.c_int),
        "mhg_matrix_upload_range": ([vp, vp, u64, u64, vp], C.c_int),
        "mhg_matrix_download": ([vp, vp, vp], C.c_int),
        "mhg_rowmajor_to_mh": ([vp, vp, vp], C.c_int),
        "mhg_mh_to_rowmajor": ([vp, vp, vp], C.c_int),
        "mhg_rowmajor_host_to_mh": ([vp, vp], C.c_int),
        "mhg_mh_to_rowmajor_host": ([vp, vp], C.c_int),
        "mhg_synchronize": ([vp], C.c_int),
        "mhg_stream_create": ([P(vp), C.c_int], C.c_int),
        "mhg_stream_destroy": ([vp], C.c_int),
        "mhg_event_create": ([P(vp)], C.c_int),
        "mhg_event_record": ([vp, vp], C.c_int),
        "mhg_event_query": ([vp, P(C.c_int)], C.c_int),
        "mhg_event_synchronize": ([vp], C.c_int),
        "mhg_stream_wait_event": ([vp, vp], C.c_int),
        "mhg_event_destroy": ([vp], C.c_int),
        "mhg_mm": ([_View, _View, _View, C.c_int, P(Counters), vp], C.c_int),
        "mhg_mm_ex": ([_View, _View, _View, C.c_int, u32, P(Counters), vp], C.c_int),
        "mhg_plan_create_ex": ([_View, _View, _View, C.c_int, u32, P(vp)], C.c_int),
        "mhg_counters_oblivious": ([_View, _View, _View, P(Counters)], C.c_int),
        "mhg_counters_layout": ([u64] * 8 + [P(Counters)], C.c_int),
        "mhg_counters_for": ([u32, _View, _View, _View, P(Counters)], C.c_int),
        "mhg_counters_geometry": ([u32] + [u64] * 12 + [P(Counters)], C.c_int),
        "mhg_plan_create": ([_View, _View, _View, C.c_int, P(vp)], C.c_int),
        "mhg_plan_run": ([vp, vp], C.c_int),
        "mhg_plan_pack": ([vp, C.c_int, vp], C.c_int),
        "mhg_plan_pack_buffer": ([vp, C.c_int, P(vp), P(u64)], C.c_int),
        "mhg_plan_gemm": ([vp, vp], C.c_int),
        "mhg_ipc_export": ([vp, P(IpcHandle), P(u64)], C.c_int),
        "mhg_ipc_open": ([P(IpcHandle), P(vp)], C.c_int),
        "mhg_ipc_close": ([vp], C.c_int),
        "mhg_copy_async": ([vp, vp, u64, vp], C.c_int),
        "mhg_dist_block": ([u32, u32, u64, u64, P(DistBlock)], C.c_int),
        "mhg_dist_slice": ([u32, u32, u64, P(u64), P(u64)], C.c_int),
        "mhg_dist_segment_count": ([u32, P(u32)], C.c_int),
        "mhg_dist_segment": ([u32, u32, u64, u64, u32, P(DistSegment)], C.c_int),
        "mhg_dist_plan_create": ([vp, vp, vp, C.c_int, u32, u32, u32, P(vp)], C.c_int),
        "mhg_sweep_create": ([P(vp), u32, P(vp)], C.c_int),
        "mhg_sweep_run": ([vp, vp], C.c_int),
        "mhg_sweep_macs": ([vp, P(u64)], C.c_int),
        "mhg_sweep_destroy": ([vp], C.c_int),
        "mhg_plan_counters": ([vp, P(Counters)], C.c_int),
        "mhg_verify": ([_View, _View, _View, _View, C.c_int, u32, u64, P(C.c_int), vp], C.c_int),
        "mhg_rng_create": ([u64, P(vp)], C.c_int),
        "mhg_rng_below": ([vp, u64, vp, u64], C.c_int),
        "mhg_rng_destroy": ([vp], C.c_int),
        "mhg_plan_info": ([vp, P(u64), P(u64), P(u32), P(u32), P(u64)], C.c_int),
        "mhg_plan_variant": ([vp, P(C.c_int), P(C.c_int)], C.c_int),
        "mhg_plan_destroy": ([vp], C.c_int),
        "mhg_limb_params": ([u32, P(u32), P(u32), P(u64)], C.c_int),
        "mhg_fold_level": ([u32, u64, P(u32)], C.c_int),
        "mhg_fold_level_u8": ([u32, u64, P(u32)], C.c_int),
        "mhg_plan_time_gemm": ([vp, C.c_int, vp, P(C.c_float)], C.c_int),
        "mhg_plan_set_profiling": ([vp, C.c_int], C.c_int),
        "mhg_plan_gemm_time": ([vp, P(C.c_float), P(u64)], C.c_int),
    }
    for name, (args, res) in sigs.items():
        if os.environ.get("MHG_LIB") and not hasattr(L, name):
            continue  # an older A/B build without this (diagnostic) entry point
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status: int):
    if status:
        msg = lib().mhg_last_error().decode(errors="replace")
        raise _ERR.get(status, DeviceError)(msg)


# ---------------------------------------------------------------- options
def set_option(key: int, value: int):
    """mhg_set_option: a planner choice or test hook (results are identical for every value)."""
    _check(lib().mhg_set_option(key, value))


def get_option(key: int) -> int:
    v = C.c_int64()
    _check(lib().mhg_get_option(key, C.byref(v)))
    return v.value


class options:
    """Context manager: `with options({OPT_DIGITS: 0}): ...` sets options, restores on exit."""

    def __init__(self, values: dict):
        self._values = dict(values)
        self._saved = {}

    def __enter__(self):
        for k, v in self._values.items():
            self._saved[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self._saved.items():
            set_option(k, v)
        return False


# ------------------------------------------------------------------ codec
class Layout:
    """layout.hpp:42-76: n = 2^m * t, tiles in Z order, row-major inside."""

    def __init__(self, n: int, t: int):
        _check(lib().mhg_layout_check(n, t))
        self.n, self.t = int(n), int(t)
        g = n // t
        self.grid_log2 = g.bit_length() - 1
        self.tile = t * t
        self.total = n * n

    def tdiv(self, v):
        return v // self.t

    def tmod(self, v):
        return v % self.t

    def __eq__(self, o):
        return isinstance(o, Layout) and (self.n, self.t) == (o.n, o.t)

    def __repr__(self):
        return f"Layout(n={self.n}, t={self.t})"


def encode(lay: Layout, i: int, j: int) -> int:
    z = C.c_uint64()
    _check(lib().mhg_encode(lay.n, lay.t, i, j, C.byref(z)))
    return z.value


def _extract(lay: Layout, z: int):
    i, j = C.c_uint64(), C.c_uint64()
    _check(lib().mhg_extract(lay.n, lay.t, z, C.byref(i), C.byref(j)))
    return i.value, j.value


def extract_i(lay: Layout, z: int) -> int:
    return _extract(lay, z)[0]


def extract_j(lay: Layout, z: int) -> int:
    return _extract(lay, z)[1]


class Modulus:
    """field.hpp:23-35: prime 2 <= q < 2^31."""

    def __init__(self, q: int):
        _check(lib().mhg_modulus_check(q))
        self.q = int(q)

    def __repr__(self):
        return f"Modulus({self.q})"


def limb_params(q: int):
    """(limbs, representative threshold H, max exact K per int32 chunk) for q."""
    L, H, K = C.c_uint32(), C.c_uint32(), C.c_uint64()
    _check(lib().mhg_limb_params(q, C.byref(L), C.byref(H), C.byref(K)))
    return L.value, H.value, K.value


def fold_level(q: int, k_chunk: int, unsigned_digits: bool = False) -> int:
    """Reductions per output the 2-limb epilogue uses for chunks of k_chunk."""
    lv = C.c_uint32()
    f = lib().mhg_fold_level_u8 if unsigned_digits else lib().mhg_fold_level
    _check(f(q, k_chunk, C.byref(lv)))
    return lv.value


def ipc_export(ptr: int):
    """(64-byte IPC handle of the device allocation containing ptr, ptr's offset in it)."""
    h, off = IpcHandle(), C.c_uint64()
    _check(lib().mhg_ipc_export(C.c_void_p(ptr), C.byref(h), C.byref(off)))
    return bytes(h.bytes), off.value


def ipc_open(handle: bytes) -> int:
    """Map a peer rank's allocation (handle from ipc_export) here; returns its base."""
    if len(handle) != 64:
        raise InvalidArgument("ipc_open: handle must be 64 bytes")
    h, base = IpcHandle(), C.c_void_p()
    C.memmove(h.bytes, handle, 64)
    _check(lib().mhg_ipc_open(C.byref(h), C.byref(base)))
    return base.value


def ipc_close(base: int):
    _check(lib().mhg_ipc_close(C.c_void_p(base)))


def copy_async(dst: int, src: int, nbytes: int, stream=None):
    """Device-to-device (or peer) copy on the copy engines, ordered on stream."""
    _check(lib().mhg_copy_async(C.c_void_p(dst), C.c_void_p(src), nbytes, _stream_ptr(stream)))


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(getattr(stream, "cuda_stream", stream))


# -------------------------------------------------------------- container
class Matrix:
    """matrix.hpp:13-39: device-resident n x n store in Morton-hybrid order.

    `cells()` downloads the flat store (numpy uint32); `upload(cells)` replaces
    it.  `device_ptr` exposes the device buffer (e.g. for torch interop).
    """

    def __init__(self, layout: Layout, modulus: Modulus, *, _wrap_ptr: Optional[int] = None,
                 _owner=None):
        self._h = C.c_void_p()
        if _wrap_ptr is None:
            _check(lib().mhg_matrix_create(layout.n, layout.t, modulus.q, C.byref(self._h)))
        else:
            _check(lib().mhg_matrix_wrap(layout.n, layout.t, modulus.q, C.c_void_p(_wrap_ptr),
                                         C.byref(self._h)))
        self._owner = _owner  # keeps a wrapped torch tensor alive
        self._layout, self._mod = layout, modulus
        ptr = C.c_void_p()
        _check(lib().mhg_matrix_info(self._h, None, None, None, C.byref(ptr)))
        self.device_ptr = ptr.value

    @classmethod
    def wrap(cls, layout: Layout, modulus: Modulus, device_ptr: int, owner=None) -> "Matrix":
        """Non-owning container over an existing device buffer of n*n uint32."""
        return cls(layout, modulus, _wrap_ptr=device_ptr, _owner=owner)

    def layout(self) -> Layout:
        return self._layout

    def modulus(self) -> Modulus:
        return self._mod

    @property
    def handle(self):
        return self._h

    def cells(self, stream=None) -> np.ndarray:
        out = np.empty(self._layout.total, dtype=np.uint32)
        _check(lib().mhg_matrix_download(self._h, out.ctypes.data, _stream_ptr(stream)))
        if stream is not None:
            import torch  # synchronise the caller's stream before reading host memory
            torch.cuda.synchronize()
        return out

    def upload(self, cells: np.ndarray, stream=None) -> "Matrix":
        a = np.ascontiguousarray(cells, dtype=np.uint32).reshape(-1)
        if a.size != self._layout.total:
            raise InvalidArgument("upload: expected n*n cells")
        _check(lib().mhg_matrix_upload(self._h, a.ctypes.data, _stream_ptr(stream)))
        if stream is not None:
            import torch
            torch.cuda.synchronize()
        return self

    @property
    def upload_bytes(self) -> int:
        """PCIe bytes moved by the last upload (2 per cell on the 16-bit wire)."""
        b = C.c_uint64()
        _check(lib().mhg_matrix_upload_bytes(self._h, C.byref(b)))
        return int(b.value)

    def at(self, i: int, j: int) -> int:
        return int(self.cells()[encode(self._layout, i, j)])

    def __eq__(self, other) -> bool:  # matrix.hpp:30-33
        return (isinstance(other, Matrix) and self._layout == other._layout
                and self._mod.q == other._mod.q
                and np.array_equal(self.cells(), other.cells()))

    def __del__(self):
        try:
            if self._h:
                lib().mhg_matrix_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def from_row_major(grid: np.ndarray, t: int, mod: Modulus) -> Matrix:
    """matrix.hpp:44-58, via the K1 conversion kernel (device)."""
    import torch
    g = np.ascontiguousarray(grid, dtype=np.uint32)
    if g.ndim != 2 or g.shape[0] != g.shape[1]:
        raise InvalidArgument("from_row_major: grid is not square")
    n = g.shape[0]
    lay = Layout(n, t)
    m = Matrix(lay, mod)
    dev = torch.from_numpy(g.view(np.int32)).cuda()
    # on torch's current stream: the buffer came from its caching allocator
    _check(lib().mhg_rowmajor_to_mh(m.handle, dev.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return m


def to_row_major(m: Matrix) -> np.ndarray:
    """matrix.hpp:60-67, via the K1 conversion kernel (device)."""
    import torch
    n = m.layout().n
    dev = torch.empty(n * n, dtype=torch.int32, device="cuda")
    # on torch's current stream, which orders the write after earlier users of the block
    _check(lib().mhg_mh_to_rowmajor(m.handle, dev.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return dev.cpu().numpy().view(np.uint32).reshape(n, n)


# ------------------------------------------------------------------ views
@dataclass
class Sub:
    """submatrix.hpp:13-18: (container, flat origin, rows, cols)."""

    mat: Optional[Matrix]
    origin: int = 0
    rows: int = 0
    cols: int = 0

    def _c(self) -> _View:
        return _View(self.mat.handle if self.mat is not None else None, self.origin, self.rows,
                     self.cols)


@dataclass
class Problem:
    """multiply.hpp:49-53: a (output) += b (left) * c (right)."""

    a: Sub
    b: Sub
    c: Sub


ALLOW_ALIAS = 1
KERNEL_NAIVE = 2    # MHG_KERNEL_NAIVE: mm_naive's validation + Counters (multiply.hpp:269-278)
KERNEL_DEFAULT = 4  # MHG_KERNEL_DEFAULT: mm_default's (multiply.hpp:283-291)


def mm(problem: Problem, op: int = OP_ADD, stream=None, allow_alias: bool = False,
       kernel: int = 0) -> Counters:
    """out op= lhs * rhs on the GPU (asynchronous on `stream`; None = default).

    allow_alias=True lifts the reference's distinct-container rule (the TU
    Schur update on views of one parent); snapshot semantics: C_new = C_old op
    A_old * B_old even when the views overlap.  kernel = KERNEL_NAIVE /
    KERNEL_DEFAULT applies that reference kernel's validation and Counters."""
    ctr = Counters()
    _check(lib().mhg_mm_ex(problem.a._c(), problem.b._c(), problem.c._c(), op,
                           (ALLOW_ALIAS if allow_alias else 0) | kernel, C.byref(ctr),
                           _stream_ptr(stream)))
    return ctr


def mm_oblivious(problem: Problem, stream=None) -> Counters:
    """Drop-in for mh::mm_oblivious (multiply.hpp:297-308): accumulate, then
    synchronise so the result is visible like the reference's synchronous call."""
    ctr = mm(problem, OP_ADD, stream)
    import torch
    torch.cuda.synchronize()
    return ctr


def mm_naive(problem: Problem, stream=None) -> Counters:
    """mm_naive (multiply.hpp:269-278): same result, its Counters; synchronous."""
    ctr = mm(problem, OP_ADD, stream, kernel=KERNEL_NAIVE)
    import torch
    torch.cuda.synchronize()
    return ctr


def mm_default(problem: Problem, stream=None) -> Counters:
    """mm_default (multiply.hpp:283-291): same result, its Counters; synchronous."""
    ctr = mm(problem, OP_ADD, stream, kernel=KERNEL_DEFAULT)
    import torch
    torch.cuda.synchronize()
    return ctr


def counters_geometry(kernel: int, geo_out, geo_lhs, geo_rhs, rows, inner, cols) -> Counters:
    """Counters of mm_oblivious (kernel 0), mm_naive (KERNEL_NAIVE) or mm_default
    (KERNEL_DEFAULT) from raw geometry, geo_* = (n, t, flat origin) per container
    (host only, no GPU needed)."""
    ctr = Counters()
    _check(lib().mhg_counters_geometry(kernel, *geo_out, *geo_lhs, *geo_rhs, rows, inner, cols,
                                       C.byref(ctr)))
    return ctr


class Sweep:
    """mhg_sweep: a sequence of plans captured, in order, into ONE CUDA graph (include/mhg.h);
    run(stream) replays every plan's packs and GEMM with a single launch."""

    def __init__(self, plans):
        self._plans = list(plans)  # keep the plans (and their containers) alive
        self._h = C.c_void_p()
        arr = (C.c_void_p * len(self._plans))(*[pl._h for pl in self._plans])
        _check(lib().mhg_sweep_create(arr, len(self._plans), C.byref(self._h)))
        m = C.c_uint64()
        _check(lib().mhg_sweep_macs(self._h, C.byref(m)))
        self.macs = m.value

    def run(self, stream=None) -> int:
        _check(lib().mhg_sweep_run(self._h, _stream_ptr(stream)))
        return self.macs

    def __del__(self):
        try:
            if self._h:
                lib().mhg_sweep_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def dist_block(nranks: int, rank: int, n: int, t: int) -> DistBlock:
    """mhg_dist_block: the rank's block of the C-stationary Morton partition (host only)."""
    b = DistBlock()
    _check(lib().mhg_dist_block(nranks, rank, n, t, C.byref(b)))
    return b


def dist_slice(nranks: int, rank: int, n: int):
    """mhg_dist_slice: flat [begin, end) of the rank's slice of an n x n store."""
    b, e = C.c_uint64(), C.c_uint64()
    _check(lib().mhg_dist_slice(nranks, rank, n, C.byref(b), C.byref(e)))
    return b.value, e.value


def dist_segments(nranks: int, rank: int, n: int, t: int):
    """mhg_dist_segment for every K segment of the rank's update (host only)."""
    cnt = C.c_uint32()
    _check(lib().mhg_dist_segment_count(nranks, C.byref(cnt)))
    out = []
    for i in range(cnt.value):
        g = DistSegment()
        _check(lib().mhg_dist_segment(nranks, rank, n, t, i, C.byref(g)))
        out.append(g)
    return out


def verify(problem: Problem, old: Sub, op: int = OP_ADD, rounds: int = 2, seed: int = 0x5EED,
           stream=None) -> bool:
    """Freivalds check on the device that problem.a now holds old op b*c (mhg_verify);
    `old` is a view (own container) of the output's cells before the multiply."""
    ok = C.c_int()
    _check(lib().mhg_verify(problem.a._c(), old._c(), problem.b._c(), problem.c._c(), op, rounds, seed,
                            C.byref(ok), _stream_ptr(stream)))
    return bool(ok.value)


class Rng:
    """mh::Rng (bench.hpp:44-52): mt19937_64(seed); below(k, count) returns the next
    `count` draws of below(k) as uint32 (the gen_problem fill order, :101-103)."""

    def __init__(self, seed: int):
        self._h = C.c_void_p()
        _check(lib().mhg_rng_create(seed, C.byref(self._h)))

    def below(self, k: int, count: int = 1, out: Optional[np.ndarray] = None) -> np.ndarray:
        a = np.empty(count, dtype=np.uint32) if out is None else out
        if a.dtype != np.uint32 or not a.flags.c_contiguous or a.size != count:
            raise InvalidArgument("Rng.below: out must be a contiguous uint32 array of count cells")
        _check(lib().mhg_rng_below(self._h, k, a.ctypes.data, count))
        return a

    def __del__(self):
        try:
            if self._h:
                lib().mhg_rng_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def counters_oblivious(problem: Problem) -> Counters:
    ctr = Counters()
    _check(lib().mhg_counters_oblivious(problem.a._c(), problem.b._c(), problem.c._c(),
                                        C.byref(ctr)))
    return ctr


def counters_layout(n, t, out_origin, lhs_origin, rhs_origin, rows, inner, cols) -> Counters:
    """Planner Counters from raw geometry (host only, no GPU needed)."""
    ctr = Counters()
    _check(lib().mhg_counters_layout(n, t, out_origin, lhs_origin, rhs_origin, rows, inner, cols,
                                     C.byref(ctr)))
    return ctr


class Plan:
    """Planned multiply replayed as one CUDA graph (pack lhs, pack rhs, GEMM)."""

    def __init__(self, problem: Problem, op: int = OP_ADD, allow_alias: bool = False):
        self._h = C.c_void_p()
        self._problem = problem  # keep containers alive
        _check(lib().mhg_plan_create_ex(problem.a._c(), problem.b._c(), problem.c._c(), op,
                                        ALLOW_ALIAS if allow_alias else 0, C.byref(self._h)))

    @classmethod
    def for_segment(cls, out: "Matrix", lhs: "Matrix", rhs: "Matrix", op: int, nranks: int,
                    rank: int, index: int) -> "Plan":
        """mhg_dist_plan_create: rank `rank`'s plan of K segment `index` of the multi-GPU
        partition over `nranks` ranks (C[R_r, C_r] op= A[R_r, k0:k1] B[k0:k1, C_r])."""
        self = cls.__new__(cls)
        self._h = C.c_void_p()
        self._problem = (out, lhs, rhs)  # keep containers alive
        _check(lib().mhg_dist_plan_create(out.handle, lhs.handle, rhs.handle, op, nranks, rank,
                                          index, C.byref(self._h)))
        return self

    def run(self, stream=None):
        _check(lib().mhg_plan_run(self._h, _stream_ptr(stream)))

    # -- split execution (multi-GPU packed-panel exchange, see dist.rank_update_packed)
    def pack(self, which: int, stream=None):
        """Pack the lhs (0) or rhs (1) view into this plan's workspace."""
        _check(lib().mhg_plan_pack(self._h, which, _stream_ptr(stream)))

    def pack_region(self, which: int):
        """(device pointer, bytes) of the packed lhs (0) / rhs (1) in the workspace."""
        ptr, nb = C.c_void_p(), C.c_uint64()
        _check(lib().mhg_plan_pack_buffer(self._h, which, C.byref(ptr), C.byref(nb)))
        return (ptr.value or 0), nb.value

    def pack_buffer(self, which: int):
        """The packed lhs (0) / rhs (1) bytes as a zero-copy uint8 CUDA tensor view of
        the plan's workspace (valid while the plan lives); plans of equal geometry
        share its layout, so it can be broadcast between ranks."""
        import torch
        ptr, nb = C.c_void_p(), C.c_uint64()
        _check(lib().mhg_plan_pack_buffer(self._h, which, C.byref(ptr), C.byref(nb)))

        class _Buf:  # __cuda_array_interface__ v3 wrapper for torch.as_tensor
            def __init__(self, p, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1",
                                                 "data": (p, False), "version": 3}
        if not nb.value:
            return torch.empty(0, dtype=torch.uint8, device="cuda")
        return torch.as_tensor(_Buf(ptr.value, nb.value), device="cuda")

    def gemm(self, stream=None):
        """The GEMM + epilogue on the current packs (no packing)."""
        _check(lib().mhg_plan_gemm(self._h, _stream_ptr(stream)))

    def counters(self) -> Counters:
        c = Counters()
        _check(lib().mhg_plan_counters(self._h, C.byref(c)))
        return c

    def info(self) -> dict:
        la, ti, li, ch, wb = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        _check(lib().mhg_plan_info(self._h, C.byref(la), C.byref(ti), C.byref(li), C.byref(ch),
                                   C.byref(wb)))
        ud, cg = C.c_int(), C.c_int()
        _check(lib().mhg_plan_variant(self._h, C.byref(ud), C.byref(cg)))
        return {"launches": la.value, "tiles": ti.value, "limbs": li.value, "k_chunks": ch.value,
                "workspace_bytes": wb.value, "digits": "u8" if ud.value else "s8",
                "cta_group": cg.value}

    def time_gemm(self, iters: int = 10, stream=None) -> float:
        ms = C.c_float()
        _check(lib().mhg_plan_time_gemm(self._h, iters, _stream_ptr(stream), C.byref(ms)))
        return ms.value

    def set_profiling(self, enable: bool = True):
        _check(lib().mhg_plan_set_profiling(self._h, int(enable)))

    def gemm_time(self):
        """(summed GEMM ms, GEMM launches) since the last call (profiling mode)."""
        ms, n = C.c_float(), C.c_uint64()
        _check(lib().mhg_plan_gemm_time(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def __del__(self):
        try:
            if self._h:
                lib().mhg_plan_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass

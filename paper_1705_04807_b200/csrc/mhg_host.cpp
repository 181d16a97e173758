// mhg_host.cpp -- implementation of the C ABI declared in include/mhg.h.
//
// Host responsibilities: validation with the reference's error classes,
// container handles, the planner (closed-form Counters + task grid), the
// packing workspace and CUDA-graph capture of a plan.  All arithmetic runs in
// the sm_100a kernels of mhg_kernels.cu; there is no CPU compute path.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <random>
#include <stdexcept>
#include <memory>
#include <string>
#include <vector>

#include "mhg.h"
#include "mhg_internal.hpp"
#include "mhg_planner.hpp"

struct mhg_matrix_s {
    uint64_t n = 0, t = 0;
    uint32_t q = 0;
    uint32_t* cells = nullptr;  // device, n*n
    bool owned = false;
    int device = 0;
    uint16_t* wire16 = nullptr;   // device scratch of the 16-bit upload wire (mhg_wire.cpp)
    uint64_t upload_bytes = 0;    // PCIe bytes of the last mhg_matrix_upload
};

namespace {

thread_local std::string g_last_error;

struct Failure {
    mhg_status code;
    std::string msg;
};

[[noreturn]] void fail(mhg_status code, const std::string& msg) { throw Failure{code, msg}; }

void cuda_check(int err, const char* what) {
    if (err != 0)
        fail(MHG_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString((cudaError_t)err));
}

template <typename F>
mhg_status guarded(F&& f) {
    try {
        f();
        return MHG_OK;
    } catch (const Failure& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return MHG_ERR_DEVICE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return MHG_ERR_DEVICE;
    }
}

// ----------------------------------------------------------------- device
// Per-device state: the properties check and the kernels' one-time attributes
// (dynamic shared memory opt-in) apply to the device that is current when they run,
// so each device gets its own, on first use.
constexpr int kMaxDevices = 64;

struct DeviceInfo {
    int sms = 0;
    bool ok = false;
    std::string why;
    std::once_flag once;
};

int current_device() {
    int dev = -1;
    const cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return dev;
}

const DeviceInfo& device_info() {
    static DeviceInfo table[kMaxDevices];
    static DeviceInfo none;
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) {
        static std::once_flag once;
        std::call_once(once, [] { none.why = "no CUDA device"; });
        return none;
    }
    DeviceInfo& info = table[dev];
    std::call_once(info.once, [&info, dev] {
        cudaDeviceProp prop{};
        const cudaError_t e = cudaGetDeviceProperties(&prop, dev);
        if (e != cudaSuccess) {
            info.why = std::string("cudaGetDeviceProperties: ") + cudaGetErrorString(e);
            return;
        }
        if (prop.major != 10 || prop.minor != 0) {
            info.why = "device " + std::string(prop.name) + " is sm_" + std::to_string(prop.major) +
                       std::to_string(prop.minor) + "; this build only runs on sm_100 (B200)";
            return;
        }
        info.sms = prop.multiProcessorCount;
        const int ce = mhg::configure_kernels();
        if (ce != 0) {
            info.why = std::string("kernel configuration: ") + cudaGetErrorString((cudaError_t)ce);
            return;
        }
        info.ok = true;
    });
    return info;
}

void require_device() {
    const DeviceInfo& d = device_info();
    if (!d.ok) fail(MHG_ERR_DEVICE, d.why);
}

// --------------------------------------------------------------- validation
// submatrix.hpp:43-51
mhg::Rect check_view(const mhg_view& v) {
    if (v.mat == nullptr) fail(MHG_ERR_INVALID_ARGUMENT, "sub-matrix: null container");
    const uint64_t n = v.mat->n, t = v.mat->t;
    if (v.origin >= n * n) fail(MHG_ERR_OUT_OF_RANGE, "sub-matrix: origin outside the container");
    const uint64_t i = mhg::extract_i(t, v.origin), j = mhg::extract_j(t, v.origin);
    if (i + v.rows > n || j + v.cols > n)
        fail(MHG_ERR_OUT_OF_RANGE, "sub-matrix: extends past the container edge");
    return mhg::Rect{i, j, v.rows, v.cols};
}

bool overlap(const mhg_matrix_s* a, const mhg_matrix_s* b) {
    const uintptr_t a0 = (uintptr_t)a->cells, a1 = a0 + a->n * a->n * 4;
    const uintptr_t b0 = (uintptr_t)b->cells, b1 = b0 + b->n * b->n * 4;
    return a0 < b1 && b0 < a1;
}

struct Checked {
    mhg::Rect ro, rl, rr;
};

// check_problem (multiply.hpp:55-66) + mm_oblivious's layout guard (:299-301); mm_naive
// and mm_default have no layout guard (their containers may differ in n and t).
Checked check_problem(const mhg_view& out, const mhg_view& lhs, const mhg_view& rhs,
                      bool allow_alias = false, bool layout_guard = true) {
    Checked c{check_view(out), check_view(lhs), check_view(rhs)};
    const bool shared = out.mat == lhs.mat || out.mat == rhs.mat || lhs.mat == rhs.mat ||
                        overlap(out.mat, lhs.mat) || overlap(out.mat, rhs.mat) ||
                        overlap(lhs.mat, rhs.mat);
    if (shared && !allow_alias)
        fail(MHG_ERR_LOGIC, "problem: the three views must live in distinct matrices");
    if (out.rows != lhs.rows || out.cols != rhs.cols || lhs.cols != rhs.rows)
        fail(MHG_ERR_LOGIC, "problem: view shapes do not chain");
    if (out.mat->q != lhs.mat->q || out.mat->q != rhs.mat->q)
        fail(MHG_ERR_LOGIC, "problem: operands use different moduli");
    if (layout_guard && (out.mat->n != lhs.mat->n || out.mat->n != rhs.mat->n ||
                         out.mat->t != lhs.mat->t || out.mat->t != rhs.mat->t))
        fail(MHG_ERR_LOGIC, "mm_oblivious: operands must share layout parameters");
    return c;
}

// Counters of the reference kernel named by flags (MHG_KERNEL_NAIVE / _DEFAULT; else
// mm_oblivious), all in closed form.
mhg::Counters counters_of(const mhg_view& out, const mhg_view& lhs, const mhg_view& rhs,
                          const Checked& c, uint32_t flags = 0) {
    if (flags & (MHG_KERNEL_NAIVE | MHG_KERNEL_DEFAULT)) {
        const mhg::Kernel3 g{{out.mat->n, out.mat->t, c.ro.i, c.ro.j},
                             {lhs.mat->n, lhs.mat->t, c.rl.i, c.rl.j},
                             {rhs.mat->n, rhs.mat->t, c.rr.i, c.rr.j},
                             c.ro.rows, c.rl.cols, c.ro.cols};
        return (flags & MHG_KERNEL_NAIVE) ? mhg::naive_counters(g) : mhg::default_counters(g);
    }
    return mhg::oblivious_counters(out.mat->n, out.mat->t, c.ro, c.rl, c.rr);
}

bool layout_guarded(uint32_t flags) { return !(flags & (MHG_KERNEL_NAIVE | MHG_KERNEL_DEFAULT)); }

void check_flags(uint32_t flags) {
    if (flags & ~(MHG_ALLOW_ALIAS | MHG_KERNEL_NAIVE | MHG_KERNEL_DEFAULT))
        fail(MHG_ERR_INVALID_ARGUMENT, "mm: unknown flag");
    if ((flags & MHG_KERNEL_NAIVE) && (flags & MHG_KERNEL_DEFAULT))
        fail(MHG_ERR_INVALID_ARGUMENT, "mm: MHG_KERNEL_NAIVE and MHG_KERNEL_DEFAULT are exclusive");
}

void put_counters(const mhg::Counters& c, mhg_counters* dst) {
    if (!dst) return;
    dst->base_case_calls = c.base_case_calls;
    dst->scalar_macs = c.scalar_macs;
    dst->encode_calls = c.encode_calls;
    dst->recursive_calls = c.recursive_calls;
    dst->max_consecutive_jump = c.max_consecutive_jump;
}

// ---------------------------------------------------------------- execution
// Device memory of one multiply: six offset tables (the coalesced epilogue
// computes output offsets in-kernel; row-per-thread epilogues, the SET fill and
// the packs read tables) and the two packed operands.
struct Buffers {
    uint64_t *out_row = nullptr, *out_col = nullptr, *lhs_row = nullptr, *lhs_col = nullptr,
             *rhs_row = nullptr, *rhs_col = nullptr;
    int8_t *apack = nullptr, *bpack = nullptr;
};

uint64_t align256(uint64_t v) { return (v + 255) & ~uint64_t(255); }

uint64_t buffer_bytes(const Checked& c, const mhg::GemmGeometry& g) {
    const uint64_t r = c.ro.rows, k = c.rl.cols, cc = c.ro.cols;
    return align256(8 * r) + align256(8 * cc) + align256(8 * r) + align256(8 * k) + align256(8 * k) +
           align256(8 * cc) + align256(g.apack_bytes) + align256(g.bpack_bytes);
}

Buffers carve(uint8_t* base, const Checked& c, const mhg::GemmGeometry& g) {
    const uint64_t r = c.ro.rows, k = c.rl.cols, cc = c.ro.cols;
    Buffers b;
    uint8_t* p = base;
    auto take = [&](uint64_t bytes) {
        uint8_t* q = p;
        p += align256(bytes);
        return q;
    };
    b.out_row = (uint64_t*)take(8 * r);
    b.out_col = (uint64_t*)take(8 * cc);
    b.lhs_row = (uint64_t*)take(8 * r);
    b.lhs_col = (uint64_t*)take(8 * k);
    b.rhs_row = (uint64_t*)take(8 * k);
    b.rhs_col = (uint64_t*)take(8 * cc);
    b.apack = (int8_t*)take(g.apack_bytes);
    b.bpack = (int8_t*)take(g.bpack_bytes);
    return b;
}

// Offset tables of the three views, each in its own container's layout.
void launch_offsets_all(const Buffers& b, const Checked& c, const mhg_view& out, const mhg_view& lhs,
                        const mhg_view& rhs, void* stream) {
    const mhg::TileGeom go = mhg::tile_geom(out.mat->t), gl = mhg::tile_geom(lhs.mat->t),
                        gr = mhg::tile_geom(rhs.mat->t);
    cuda_check(mhg::launch_offsets(b.out_row, c.ro.i, c.ro.rows, go, 1, stream), "offsets");
    cuda_check(mhg::launch_offsets(b.out_col, c.ro.j, c.ro.cols, go, 0, stream), "offsets");
    cuda_check(mhg::launch_offsets(b.lhs_row, c.rl.i, c.rl.rows, gl, 1, stream), "offsets");
    cuda_check(mhg::launch_offsets(b.lhs_col, c.rl.j, c.rl.cols, gl, 0, stream), "offsets");
    cuda_check(mhg::launch_offsets(b.rhs_row, c.rr.i, c.rr.rows, gr, 1, stream), "offsets");
    cuda_check(mhg::launch_offsets(b.rhs_col, c.rr.j, c.rr.cols, gr, 0, stream), "offsets");
}

mhg::GemmParams gemm_params(const Buffers& b, const mhg_view& out, const Checked& c,
                            const mhg::GemmGeometry& g, mhg_op op) {
    const uint32_t q = out.mat->q;
    mhg::GemmParams p{};
    p.apack = b.apack;
    p.bpack = b.bpack;
    p.out = out.mat->cells;
    p.out_rowoff = b.out_row;
    p.out_coloff = b.out_col;
    p.rows = c.ro.rows;
    p.cols = c.ro.cols;
    p.out_i0 = c.ro.i;
    p.out_j0 = c.ro.j;
    p.out_geom = mhg::tile_geom(out.mat->t);
    p.Mt = g.Mt;
    p.Nt = g.Nt;
    p.Kt = g.Kt;
    p.KC = g.KC;
    p.q = q;
    p.w32 = (uint32_t)((uint64_t(1) << 32) % q);
    p.mu = ~uint64_t(0) / q;
    const uint64_t two62 = uint64_t(1) << 62;
    p.bias = ((two62 + q - 1) / q) * q;
    p.m32 = (uint32_t)((uint64_t(1) << 32) / q);
    p.nq = (uint32_t)(0u - q);
    p.bias32 = (uint32_t)(((uint64_t(1) << 31) / q) * q);
    p.w16 = (uint32_t)((uint64_t(1) << 16) % q);
    p.w16_small = p.w16 < 256;
    p.udig = g.udig ? 1 : 0;
    // cheapest exact fold for the longest chunk; u8 digits: non-negative class sums, no
    // bias, levels from the u8 bounds.  MHG_OPT_MIN_FOLD_LEVEL only raises the level.
    const uint64_t kchunk = (uint64_t)std::min(g.Kt, g.KC) * mhg::kBK;
    if (g.udig) p.bias32 = 0;
    p.fold = g.L != 2 ? 3 : (g.udig ? mhg::fold_level_u8(q, kchunk) : mhg::fold_level(q, kchunk));
    p.fold = std::max<int>(p.fold, (int)mhg::option(mhg::kOptMinFold));
    // raster group (row tiles sharing rhs panels in L2): 8 measured best up to n = 16384
    // (profiles/r01_raster_groups.txt; G = 4 / 6 / 12 within noise or slower), 4 from 256
    // column tiles on (n = 32768: 95.4 vs 97.0 ms, G = 12 108 ms; profiles/r02_raster_groups.txt)
    p.group = g.Nt >= 256 ? 4 : 8;
    // short K: both packed operands fit in L2 with room to spare, so the rhs stages are kept
    // too (the C stream is evict-first) instead of streamed (long K: 4 MB rhs panels, each
    // needed by one raster group only)
    p.keep_b = g.apack_bytes + g.bpack_bytes <= (uint64_t(80) << 20) ? 1 : 0;
    p.narrow = g.narrow ? 1 : 0;
    // suspend (instead of re-polling) in mbarrier waits: -1% at n = 16384 / 8192 under the
    // power cap (profiles/r01_wait_hint.txt); the thread wakes when the phase completes
    p.wait_hint = 100000;
    p.mode = op == MHG_OP_SET ? 2 : 0;
    p.vec_ok = out.mat->t % 4 == 0;
    return p;
}

// 2D uint8 tensor map over a packed operand: rows of kBK bytes, box of
// `box_rows` rows, no swizzle (the pack kernels already wrote the swizzled
// shared-memory image).  cuTensorMapEncodeTiled comes from the driver entry
// point, so the library does not link libcuda.
struct TensorMaps {
    CUtensorMap a, b;
};

// 2D tiled tensor map, no swizzle: dims {d0 (inner), d1}, row pitch `pitch` bytes.
void encode_2d(CUtensorMap* tm, CUtensorMapDataType dtype, const void* base, uint64_t d0, uint64_t d1,
               uint64_t pitch, uint32_t b0, uint32_t b1) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
                   "cuTensorMapEncodeTiled lookup");
        if (!fn || q != cudaDriverEntryPointSuccess)
            fail(MHG_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<Encode>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)d0, (cuuint64_t)d1};
    const cuuint64_t strides[1] = {(cuuint64_t)pitch};
    const cuuint32_t box[2] = {b0, b1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(tm, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(MHG_ERR_DEVICE, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// Packed operand: rows of kBK bytes, boxes of `box_rows` rows.
void make_tmap(CUtensorMap* tm, const void* base, uint64_t bytes, uint32_t box_rows) {
    encode_2d(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, mhg::kBK, bytes / mhg::kBK, mhg::kBK,
              (uint32_t)mhg::kBK, box_rows);
}

// K1 conversions: the TMA kernel (default; MHG_CONV=1/2 select the LDG/STG kernels)
// for power-of-two 4 <= t <= 256 with 16-byte aligned rows, else the LDG/STG kernels.
void convert(const mhg_matrix_s* m, uint32_t* rows, int to_mh, int* flag, void* stream) {
    const int64_t mode = mhg::option(mhg::kOptConvKernel);  // 0 TMA, 1 Morton LDG/STG, 2 row-order
    const mhg::TileGeom g = mhg::tile_geom(m->t);
    const bool tma = mode == 0 && g.shift >= 0 && m->t % 4 == 0 && m->t <= 256 && m->n % 4 == 0 &&
                     m->n < (uint64_t(1) << 31) && ((uintptr_t)rows & 15) == 0;
    if (tma) {
        CUtensorMap tm;
        encode_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, rows, m->n, m->n, m->n * 4, (uint32_t)m->t,
                  mhg::conv_tma_box_rows(m->t));
        cuda_check(mhg::launch_conv_tma(&tm, m->cells, m->n, g, m->q, flag, to_mh, device_info().sms,
                                        stream),
                   to_mh ? "rowmajor_to_mh" : "mh_to_rowmajor");
    } else if (to_mh) {
        cuda_check(mhg::launch_rm_to_mh(rows, m->cells, m->n, g, m->q, flag, mode <= 1, stream),
                   "rowmajor_to_mh");
    } else {
        cuda_check(mhg::launch_mh_to_rm(m->cells, rows, m->n, g, mode <= 1, stream), "mh_to_rowmajor");
    }
}

TensorMaps tensor_maps(const Buffers& b, const mhg::GemmGeometry& g) {
    TensorMaps t{};
    if (g.pair) {
        make_tmap(&t.a, b.apack, g.apack_bytes, mhg::kBM);
        make_tmap(&t.b, b.bpack, g.bpack_bytes, (uint32_t)mhg::gemm2_b_box_rows((int)g.L));
    }
    return t;
}

void launch_gemm_any(const mhg::GemmParams& p, const mhg::GemmGeometry& g, const TensorMaps& tm,
                     void* stream) {
    if (g.pair)
        cuda_check(mhg::launch_gemm2((int)g.L, p, &tm.a, &tm.b, device_info().sms, stream), "gemm2");
    else
        cuda_check(mhg::launch_gemm((int)g.L, p, device_info().sms, stream), "gemm");
}

// Pack job of one operand (which = 0: lhs, K-major rows, digits negated for C -= A.B;
// 1: rhs, transposed).
mhg::PackArgs pack_args(const Buffers& b, const mhg_view& out, const mhg_view& v, const Checked& c,
                        const mhg::GemmGeometry& g, mhg_op op, int which) {
    const mhg::LimbParams lp = mhg::limb_params(out.mat->q);
    mhg::PackArgs a{};
    a.src = v.mat->cells;
    a.vecok = v.mat->t % 4 == 0;  // 16-byte runs inside the source's tile rows
    a.Kt = g.Kt;
    if (which == 0) {
        a.rowoff = b.lhs_row;
        a.coloff = b.lhs_col;
        a.R = c.rl.rows;
        a.K = c.rl.cols;
        a.rpt = mhg::kBM;
        a.Rtiles = g.Mt;
        a.dst = b.apack;
        a.dp = mhg::DigitParams{out.mat->q, lp.H, op == MHG_OP_SUB ? 1 : 0, g.udig ? 1 : 0};
    } else {
        a.rowoff = b.rhs_row;
        a.coloff = b.rhs_col;
        a.R = c.rr.cols;
        a.K = c.rr.rows;
        a.rpt = g.W;
        a.Rtiles = g.Nt;
        a.dst = b.bpack;
        a.dp = mhg::DigitParams{out.mat->q, lp.H, 0, g.udig ? 1 : 0};
    }
    return a;
}

void launch_pack_operand(const Buffers& b, const mhg_view& out, const mhg_view& v, const Checked& c,
                         const mhg::GemmGeometry& g, mhg_op op, int which, void* stream) {
    const mhg::PackArgs a = pack_args(b, out, v, c, g, op, which);
    cuda_check(mhg::launch_pack((int)g.L, which, a.src, a.rowoff, a.coloff, a.vecok, a.R, a.K, a.rpt,
                                a.Rtiles, a.Kt, a.dst, a.dp, stream),
               which == 0 ? "pack lhs" : "pack rhs");
}

void launch_gemm_stage(const Buffers& b, const mhg_view& out, const Checked& c,
                       const mhg::GemmGeometry& g, mhg_op op, void* stream,
                       cudaEvent_t gemm_begin = nullptr, cudaEvent_t gemm_end = nullptr);

// Pack both operands (one k_pack_pair launch: two HBM-bound grids would pay two
// ramp-down tails, profiles/r01_pack_fused.txt) and run the GEMM.
void launch_multiply(const Buffers& b, const mhg_view& out, const mhg_view& lhs,
                     const mhg_view& rhs, const Checked& c, const mhg::GemmGeometry& g,
                     mhg_op op, void* stream, cudaEvent_t gemm_begin = nullptr,
                     cudaEvent_t gemm_end = nullptr) {
    cuda_check(mhg::launch_pack_pair((int)g.L, pack_args(b, out, lhs, c, g, op, 0),
                                     pack_args(b, out, rhs, c, g, op, 1), stream),
               "pack lhs + rhs");
    launch_gemm_stage(b, out, c, g, op, stream, gemm_begin, gemm_end);
}

// The GEMM on the current packs (+ the opt-in MHG_OPT_GEMM_STATS report).
void launch_gemm_stage(const Buffers& b, const mhg_view& out, const Checked& c,
                       const mhg::GemmGeometry& g, mhg_op op, void* stream, cudaEvent_t gemm_begin,
                       cudaEvent_t gemm_end) {
    mhg::GemmParams p = gemm_params(b, out, c, g, op);
    // diagnostics: MHG_OPT_GEMM_STATS = 1 prints per-CTA wait-cycle shares (synchronous)
    const bool stats_on = mhg::option(mhg::kOptGemmStats) != 0 && mhg::diag_build();
    struct StatsBuf {  // freed on every path, including a failed launch
        unsigned long long* ptr = nullptr;
        ~StatsBuf() {
            if (ptr) cudaFree(ptr);
        }
    } statsbuf;
    unsigned long long* stats = nullptr;
    if (stats_on) {
        const size_t bytes = (size_t)device_info().sms * mhg::kStatCount * sizeof(unsigned long long);
        cuda_check(cudaMalloc(&statsbuf.ptr, bytes), "stats alloc");
        cuda_check(cudaMemset(statsbuf.ptr, 0, bytes), "stats zero");
        stats = p.stats = statsbuf.ptr;
    }
    const TensorMaps tm = tensor_maps(b, g);
    // under stream capture (the plans' profiling graph) the records must become event-record
    // nodes of the graph (cudaEventRecordExternal); outside capture that flag is refused
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (gemm_begin || gemm_end)
        cuda_check(cudaStreamIsCapturing((cudaStream_t)stream, &cst), "capture query");
    const unsigned rec_flags = cst == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (gemm_begin) cuda_check(cudaEventRecordWithFlags(gemm_begin, (cudaStream_t)stream, rec_flags), "event");
    launch_gemm_any(p, g, tm, stream);
    if (gemm_end) cuda_check(cudaEventRecordWithFlags(gemm_end, (cudaStream_t)stream, rec_flags), "event");
    if (stats) {
        const int n = device_info().sms;
        std::vector<unsigned long long> h((size_t)n * mhg::kStatCount);
        cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "stats sync");
        cuda_check(cudaMemcpy(h.data(), stats, h.size() * 8, cudaMemcpyDeviceToHost), "stats copy");
        // MMA-side counters come from MMA-issuing CTAs only (pair leaders);
        // producer / epilogue counters from every CTA: normalise separately
        double tot = 0, s[mhg::kStatCount] = {0};
        int issuers = 0;
        for (int b = 0; b < n; ++b) {
            if (h[(size_t)b * mhg::kStatCount + mhg::kStatTotal]) ++issuers;
            for (int k = 0; k < mhg::kStatCount; ++k) s[k] += (double)h[(size_t)b * mhg::kStatCount + k];
        }
        tot = s[mhg::kStatTotal] / (issuers ? issuers : 1);
        for (int k : {1, 2}) s[k] /= (issuers ? issuers : 1);
        for (int k : {3, 4, 5, 6, 7, 8, 9, 10}) s[k] /= n;
        std::fprintf(stderr,
                     "[mhg stats] L=%u tiles=%u  MMA wait(full)=%.1f%%  MMA wait(tmem_empty)=%.1f%%  "
                     "producer wait(empty)=%.1f%%  epilogue wait(tmem_full)=%.1f%%  epilogue busy=%.1f%%  "
                     "epilogue prologue=%.1f%% (issue %.1f%%, C_old landing %.1f%%)  epilogue stores=%.1f%%  "
                     "tmem ld wait=%.1f%%  "
                     "(cycles per MMA issuer %.3g, %s)\n",
                     g.L, g.Mt * g.Nt, 100 * s[1] / tot, 100 * s[2] / tot, 100 * s[3] / tot,
                     100 * s[4] / tot, 100 * s[5] / tot, 100 * s[6] / tot, 100 * s[9] / tot, 100 * s[10] / tot, 100 * s[7] / tot, 100 * s[8] / tot, tot,
                     g.pair ? "cta pair" : "1 cta");
    }
}

// One-shot workspace for mhg_mm, one per device: grows on demand; an event orders
// reuse across streams.  Growing synchronises the device, so it is refused while the
// caller's stream is being captured (plans own their workspace: mhg_plan_create).
struct Workspace {
    std::mutex mu;
    uint8_t* base = nullptr;
    uint64_t bytes = 0;
    cudaEvent_t last = nullptr;

    uint8_t* acquire(uint64_t need, void* stream) {
        if (!last) cuda_check(cudaEventCreateWithFlags(&last, cudaEventDisableTiming), "event");
        if (need > bytes) {
            cuda_check(cudaDeviceSynchronize(), "workspace sync");
            if (base) cudaFree(base);
            base = nullptr;
            bytes = 0;
            cuda_check(cudaMalloc(&base, need), "workspace alloc");
            bytes = need;
        } else {
            cuda_check(cudaStreamWaitEvent((cudaStream_t)stream, last, 0), "workspace order");
        }
        return base;
    }
    void release(void* stream) { cuda_check(cudaEventRecord(last, (cudaStream_t)stream), "event"); }
};

Workspace& workspace() {
    // leaked on purpose: no teardown-order issues with the CUDA runtime
    static Workspace* ws[kMaxDevices] = {};
    static std::mutex mu;
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) fail(MHG_ERR_DEVICE, "no CUDA device");
    std::lock_guard<std::mutex> lock(mu);
    if (!ws[dev]) ws[dev] = new Workspace();
    return *ws[dev];
}

void refuse_capture(void* stream, const char* what) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing((cudaStream_t)stream, &st), "capture query");
    if (st != cudaStreamCaptureStatusNone)
        fail(MHG_ERR_UNSUPPORTED, std::string(what) +
                                      ": not capturable (it may allocate and synchronise); capture "
                                      "mhg_plan_run of an mhg_plan_create plan instead");
}

// Containers are device allocations: every view of a call must live on the current device.
void require_resident(std::initializer_list<const mhg_matrix_s*> mats) {
    const int dev = current_device();
    for (const mhg_matrix_s* m : mats)
        if (m && m->device != dev)
            fail(MHG_ERR_INVALID_ARGUMENT, "container lives on device " + std::to_string(m->device) +
                                               ", the current device is " + std::to_string(dev));
}

}  // namespace

// ============================================================ plan object
struct mhg_plan_s {
    mhg_view out{}, lhs{}, rhs{};
    mhg_op op = MHG_OP_ADD;
    Checked chk{};
    mhg::GemmGeometry geo{};
    mhg::Counters ctr{};
    uint8_t* mem = nullptr;
    uint64_t mem_bytes = 0;
    Buffers buf{};
    bool empty = false;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    // profiling: event pairs bracketing each GEMM launch (ring, read + reset)
    bool profiling = false;
    std::vector<cudaEvent_t> ev;
    size_t ev_used = 0;
    // profiling graph: the plan's graph with event-record nodes around the GEMM; every run
    // points the two nodes at the next ring pair, so profiled runs cost one graph launch
    // (no per-kernel host launches between the steps of a timed loop)
    cudaGraph_t pgraph = nullptr;
    cudaGraphExec_t pexec = nullptr;
    cudaGraphNode_t pnode[2] = {nullptr, nullptr};
    cudaEvent_t pev[2] = {nullptr, nullptr};
};

struct mhg_sweep_s {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t macs = 0;
    uint32_t steps = 0;
};

namespace {
// Capture fn(stream) into a graph on a private capturing stream.
template <typename F>
cudaGraph_t capture_graph(F&& fn) {
    cudaStream_t cap;
    cuda_check(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
    cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "capture");
    try {
        fn(cap);
    } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(cap, &g);
        if (g) cudaGraphDestroy(g);
        cudaStreamDestroy(cap);
        throw;
    }
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamEndCapture(cap, &g), "end capture");
    cudaStreamDestroy(cap);
    return g;
}
}  // namespace

extern "C" {

const char* mhg_last_error(void) { return g_last_error.c_str(); }

const char* mhg_version(void) { return "mhg 0.2 (sm_100a tcgen05 kind::i8)"; }

mhg_status mhg_set_option(int key, int64_t value) {
    return guarded([&] {
        if (!mhg::option_valid(key, value))
            fail(MHG_ERR_INVALID_ARGUMENT, "set_option: unknown key or value out of range");
        if (key == mhg::kOptGemmStats && value && !mhg::diag_build())
            fail(MHG_ERR_UNSUPPORTED, "set_option: GEMM wait-cycle counters are compiled only into "
                                      "diagnostic builds (-DMHG_DIAG=1, profiles/build_variant.sh)");
        mhg::set_option(key, value);
    });
}

mhg_status mhg_get_option(int key, int64_t* value) {
    return guarded([&] {
        if (!value || key <= 0 || key >= mhg::kOptCount)
            fail(MHG_ERR_INVALID_ARGUMENT, "get_option: unknown key or null output");
        *value = mhg::option(key);
    });
}

mhg_status mhg_device_check(void) {
    return guarded([] { require_device(); });
}

mhg_status mhg_layout_check(uint64_t n, uint64_t t) {
    return guarded([&] {
        if (t == 0 || n == 0) fail(MHG_ERR_INVALID_ARGUMENT, "Layout: side lengths must be positive");
        if (n >= (uint64_t(1) << 32))
            fail(MHG_ERR_INVALID_ARGUMENT, "Layout: side too large for one-word indices");
        if (!mhg::layout_ok(n, t)) fail(MHG_ERR_INVALID_ARGUMENT, "Layout: n must equal t * 2^m");
    });
}

mhg_status mhg_modulus_check(uint32_t q) {
    return guarded([&] {
        if (q < 2 || q >= (uint32_t(1) << 31))
            fail(MHG_ERR_INVALID_ARGUMENT, "Modulus: q must satisfy 2 <= q < 2^31");
        if (!mhg::is_prime(q)) fail(MHG_ERR_INVALID_ARGUMENT, "Modulus: q must be prime");
    });
}

mhg_status mhg_encode(uint64_t n, uint64_t t, uint64_t i, uint64_t j, uint64_t* z) {
    mhg_status s = mhg_layout_check(n, t);
    if (s) return s;
    return guarded([&] {
        if (i >= n || j >= n) fail(MHG_ERR_OUT_OF_RANGE, "encode: cell outside the matrix");
        *z = mhg::encode(t, i, j);
    });
}

mhg_status mhg_extract(uint64_t n, uint64_t t, uint64_t z, uint64_t* i, uint64_t* j) {
    mhg_status s = mhg_layout_check(n, t);
    if (s) return s;
    return guarded([&] {
        if (z >= n * n) fail(MHG_ERR_OUT_OF_RANGE, "extract: index outside the matrix");
        *i = mhg::extract_i(t, z);
        *j = mhg::extract_j(t, z);
    });
}

mhg_status mhg_limb_params(uint32_t q, uint32_t* limbs, uint32_t* threshold, uint64_t* k_max) {
    mhg_status s = mhg_modulus_check(q);
    if (s) return s;
    const mhg::LimbParams lp = mhg::limb_params(q);
    if (limbs) *limbs = lp.L;
    if (threshold) *threshold = lp.H;
    if (k_max) *k_max = lp.k_max;
    return MHG_OK;
}

mhg_status mhg_fold_level_u8(uint32_t q, uint64_t k_chunk, uint32_t* level) {
    mhg_status s = mhg_modulus_check(q);
    if (s) return s;
    return guarded([&] {
        if (!level) fail(MHG_ERR_INVALID_ARGUMENT, "fold_level_u8: null output");
        *level = mhg::limb_params(q).L == 2 ? (uint32_t)mhg::fold_level_u8(q, k_chunk) : 3u;
    });
}

mhg_status mhg_fold_level(uint32_t q, uint64_t k_chunk, uint32_t* level) {
    mhg_status s = mhg_modulus_check(q);
    if (s) return s;
    return guarded([&] {
        if (!level) fail(MHG_ERR_INVALID_ARGUMENT, "fold_level: null output");
        *level = mhg::limb_params(q).L == 2 ? (uint32_t)mhg::fold_level(q, k_chunk) : 3u;
    });
}

// ------------------------------------------------------------- containers
mhg_status mhg_matrix_create(uint64_t n, uint64_t t, uint32_t q, mhg_matrix* out) {
    mhg_status s = mhg_layout_check(n, t);
    if (s) return s;
    if ((s = mhg_modulus_check(q))) return s;
    return guarded([&] {
        if (!out) fail(MHG_ERR_INVALID_ARGUMENT, "matrix_create: null out");
        require_device();
        auto* m = new mhg_matrix_s();
        m->n = n;
        m->t = t;
        m->q = q;
        m->owned = true;
        cudaGetDevice(&m->device);
        const uint64_t bytes = n * n * 4;
        cudaError_t e = cudaMalloc(&m->cells, bytes);
        if (e != cudaSuccess) {
            delete m;
            cuda_check((int)e, "matrix alloc");
        }
        e = cudaMemset(m->cells, 0, bytes);
        if (e != cudaSuccess) {
            cudaFree(m->cells);
            delete m;
            cuda_check((int)e, "matrix zero");
        }
        *out = m;
    });
}

mhg_status mhg_matrix_wrap(uint64_t n, uint64_t t, uint32_t q, void* device_cells, mhg_matrix* out) {
    mhg_status s = mhg_layout_check(n, t);
    if (s) return s;
    if ((s = mhg_modulus_check(q))) return s;
    return guarded([&] {
        if (!out || !device_cells) fail(MHG_ERR_INVALID_ARGUMENT, "matrix_wrap: null pointer");
        if ((uintptr_t)device_cells % 16)
            fail(MHG_ERR_INVALID_ARGUMENT, "matrix_wrap: cells must be 16-byte aligned");
        auto* m = new mhg_matrix_s();
        m->n = n;
        m->t = t;
        m->q = q;
        m->cells = (uint32_t*)device_cells;
        m->owned = false;
        // the device that owns the buffer (the current one if the runtime cannot tell)
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, device_cells) == cudaSuccess &&
            attr.type == cudaMemoryTypeDevice)
            m->device = attr.device;
        else {
            cudaGetLastError();
            m->device = current_device();
        }
        *out = m;
    });
}

mhg_status mhg_matrix_destroy(mhg_matrix m) {
    return guarded([&] {
        if (!m) return;
        if (m->owned && m->cells) cudaFree(m->cells);
        if (m->wire16) cudaFree(m->wire16);
        delete m;
    });
}

mhg_status mhg_matrix_info(mhg_matrix m, uint64_t* n, uint64_t* t, uint32_t* q, void** cells) {
    return guarded([&] {
        if (!m) fail(MHG_ERR_INVALID_ARGUMENT, "matrix_info: null matrix");
        if (n) *n = m->n;
        if (t) *t = m->t;
        if (q) *q = m->q;
        if (cells) *cells = m->cells;
    });
}

namespace {
void upload_cells(mhg_matrix m, const uint32_t* host, uint64_t offset, uint64_t count, void* stream) {
    if (mhg::wire16_enabled(m->q, count)) {
        require_device();
        require_resident({m});  // the wire widens on the device with a kernel
        cuda_check(mhg::upload_wire16(m->cells, &m->wire16, m->n * m->n, offset, host, count,
                                      device_info().sms, stream, &m->upload_bytes),
                   "upload (16-bit wire)");
        return;
    }
    cuda_check(cudaMemcpyAsync(m->cells + offset, host, count * 4, cudaMemcpyHostToDevice,
                               (cudaStream_t)stream),
               "upload");
    m->upload_bytes = count * 4;
}
}  // namespace

mhg_status mhg_matrix_upload(mhg_matrix m, const uint32_t* host, void* stream) {
    return guarded([&] {
        if (!m || !host) fail(MHG_ERR_INVALID_ARGUMENT, "matrix_upload: null pointer");
        upload_cells(m, host, 0, m->n * m->n, stream);
    });
}

mhg_status mhg_matrix_upload_range(mhg_matrix m, const uint32_t* host, uint64_t offset,
                                   uint64_t count, void* stream) {
    return guarded([&] {
        if (!m || (!host && count)) fail(MHG_ERR_INVALID_ARGUMENT, "matrix_upload_range: null pointer");
        if (offset > m->n * m->n || count > m->n * m->n - offset)
            fail(MHG_ERR_OUT_OF_RANGE, "matrix_upload_range: cells outside the container");
        if (count) upload_cells(m, host, offset, count, stream);
    });
}

mhg_status mhg_matrix_upload_bytes(mhg_matrix m, uint64_t* bytes) {
    return guarded([&] {
        if (!m || !bytes) fail(MHG_ERR_INVALID_ARGUMENT, "matrix_upload_bytes: null pointer");
        *bytes = m->upload_bytes;
    });
}

mhg_status mhg_matrix_download(mhg_matrix m, uint32_t* host, void* stream) {
    return guarded([&] {
        if (!m || !host) fail(MHG_ERR_INVALID_ARGUMENT, "matrix_download: null pointer");
        cuda_check(cudaMemcpyAsync(host, m->cells, m->n * m->n * 4, cudaMemcpyDeviceToHost,
                                   (cudaStream_t)stream),
                   "download");
    });
}

mhg_status mhg_rowmajor_to_mh(mhg_matrix dst, const uint32_t* rows, void* stream) {
    return guarded([&] {
        if (!dst || !rows) fail(MHG_ERR_INVALID_ARGUMENT, "rowmajor_to_mh: null pointer");
        require_device();
        require_resident({dst});
        // one residue-check flag per device
        static int* flags[kMaxDevices] = {};
        static std::mutex mu;
        std::lock_guard<std::mutex> lock(mu);
        int*& flag = flags[current_device()];
        if (!flag) cuda_check(cudaMalloc(&flag, sizeof(int)), "flag alloc");
        cudaStream_t s = (cudaStream_t)stream;
        cuda_check(cudaMemsetAsync(flag, 0, sizeof(int), s), "flag");
        convert(dst, const_cast<uint32_t*>(rows), 1, flag, stream);
        int bad = 0;
        cuda_check(cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, s), "flag");
        cuda_check(cudaStreamSynchronize(s), "rowmajor_to_mh sync");
        if (bad) fail(MHG_ERR_INVALID_ARGUMENT, "from_row_major: residue out of range");
    });
}

mhg_status mhg_mh_to_rowmajor(mhg_matrix src, uint32_t* rows, void* stream) {
    return guarded([&] {
        if (!src || !rows) fail(MHG_ERR_INVALID_ARGUMENT, "mh_to_rowmajor: null pointer");
        require_device();
        require_resident({src});
        convert(src, rows, 0, nullptr, stream);
    });
}

mhg_status mhg_synchronize(void* stream) {
    return guarded([&] {
        require_device();
        cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "synchronize");
    });
}

mhg_status mhg_stream_create(void** stream, int non_blocking) {
    return guarded([&] {
        if (!stream) fail(MHG_ERR_INVALID_ARGUMENT, "stream_create: null output");
        require_device();
        cudaStream_t s = nullptr;
        cuda_check(cudaStreamCreateWithFlags(&s, non_blocking ? cudaStreamNonBlocking : cudaStreamDefault),
                   "stream create");
        *stream = s;
    });
}

mhg_status mhg_stream_destroy(void* stream) {
    return guarded([&] {
        if (!stream) return;
        cuda_check(cudaStreamDestroy((cudaStream_t)stream), "stream destroy");
    });
}

mhg_status mhg_event_create(void** event) {
    return guarded([&] {
        if (!event) fail(MHG_ERR_INVALID_ARGUMENT, "event_create: null output");
        require_device();
        cudaEvent_t e = nullptr;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
        *event = e;
    });
}

mhg_status mhg_event_record(void* event, void* stream) {
    return guarded([&] {
        if (!event) fail(MHG_ERR_INVALID_ARGUMENT, "event_record: null event");
        cuda_check(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream), "event record");
    });
}

mhg_status mhg_event_query(void* event, int* done) {
    return guarded([&] {
        if (!event || !done) fail(MHG_ERR_INVALID_ARGUMENT, "event_query: null pointer");
        const cudaError_t e = cudaEventQuery((cudaEvent_t)event);
        if (e != cudaSuccess && e != cudaErrorNotReady) cuda_check(e, "event query");
        *done = e == cudaSuccess;
    });
}

mhg_status mhg_event_synchronize(void* event) {
    return guarded([&] {
        if (!event) fail(MHG_ERR_INVALID_ARGUMENT, "event_synchronize: null event");
        cuda_check(cudaEventSynchronize((cudaEvent_t)event), "event synchronize");
    });
}

mhg_status mhg_stream_wait_event(void* stream, void* event) {
    return guarded([&] {
        if (!event) fail(MHG_ERR_INVALID_ARGUMENT, "stream_wait_event: null event");
        cuda_check(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0), "stream wait event");
    });
}

mhg_status mhg_event_destroy(void* event) {
    return guarded([&] {
        if (!event) return;
        cuda_check(cudaEventDestroy((cudaEvent_t)event), "event destroy");
    });
}

mhg_status mhg_rowmajor_host_to_mh(mhg_matrix dst, const uint32_t* host_rows) {
    return guarded([&] {
        if (!dst || !host_rows) fail(MHG_ERR_INVALID_ARGUMENT, "rowmajor_host_to_mh: null pointer");
        require_device();
        uint32_t* tmp = nullptr;
        const uint64_t bytes = dst->n * dst->n * 4;
        cuda_check(cudaMalloc(&tmp, bytes), "scratch alloc");
        mhg_status st = MHG_OK;
        const cudaError_t e = cudaMemcpy(tmp, host_rows, bytes, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) st = mhg_rowmajor_to_mh(dst, tmp, nullptr);
        const std::string msg = g_last_error;
        cudaFree(tmp);
        cuda_check((int)e, "rowmajor upload");
        if (st) fail(st, msg);
    });
}

mhg_status mhg_mh_to_rowmajor_host(mhg_matrix src, uint32_t* host_rows) {
    return guarded([&] {
        if (!src || !host_rows) fail(MHG_ERR_INVALID_ARGUMENT, "mh_to_rowmajor_host: null pointer");
        require_device();
        uint32_t* tmp = nullptr;
        const uint64_t bytes = src->n * src->n * 4;
        cuda_check(cudaMalloc(&tmp, bytes), "scratch alloc");
        int err = 0;
        try {
            convert(src, tmp, 0, nullptr, nullptr);
        } catch (...) {
            cudaFree(tmp);
            throw;
        }
        err = (int)cudaMemcpy(host_rows, tmp, bytes, cudaMemcpyDeviceToHost);
        cudaFree(tmp);
        cuda_check(err, "mh_to_rowmajor_host");
    });
}

// --------------------------------------------------------------- multiply
mhg_status mhg_counters_oblivious(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_counters* ctr) {
    return guarded([&] {
        const Checked c = check_problem(out, lhs, rhs);
        put_counters(counters_of(out, lhs, rhs, c), ctr);
    });
}

mhg_status mhg_counters_layout(uint64_t n, uint64_t t, uint64_t out_origin, uint64_t lhs_origin,
                               uint64_t rhs_origin, uint64_t rows, uint64_t inner, uint64_t cols,
                               mhg_counters* ctr) {
    return mhg_counters_geometry(0u, n, t, out_origin, n, t, lhs_origin, n, t, rhs_origin, rows, inner,
                                 cols, ctr);
}

mhg_status mhg_counters_for(uint32_t flags, mhg_view out, mhg_view lhs, mhg_view rhs, mhg_counters* ctr) {
    return guarded([&] {
        check_flags(flags);
        const Checked c = check_problem(out, lhs, rhs, false, layout_guarded(flags));
        put_counters(counters_of(out, lhs, rhs, c, flags), ctr);
    });
}

mhg_status mhg_counters_geometry(uint32_t flags, uint64_t n_out, uint64_t t_out, uint64_t out_origin,
                                 uint64_t n_lhs, uint64_t t_lhs, uint64_t lhs_origin, uint64_t n_rhs,
                                 uint64_t t_rhs, uint64_t rhs_origin, uint64_t rows, uint64_t inner,
                                 uint64_t cols, mhg_counters* ctr) {
    mhg_status s = mhg_layout_check(n_out, t_out);
    if (!s) s = mhg_layout_check(n_lhs, t_lhs);
    if (!s) s = mhg_layout_check(n_rhs, t_rhs);
    if (s) return s;
    return guarded([&] {
        check_flags(flags);
        // three distinct host-side stand-ins: only geometry is inspected
        mhg_matrix_s a, b, c;
        a.n = n_out, b.n = n_lhs, c.n = n_rhs;
        a.t = t_out, b.t = t_lhs, c.t = t_rhs;
        a.q = b.q = c.q = 2;
        a.cells = (uint32_t*)(uintptr_t)16;
        b.cells = (uint32_t*)(uintptr_t)(16 + 4 * n_out * n_out);
        c.cells = (uint32_t*)(uintptr_t)(16 + 4 * n_out * n_out + 4 * n_lhs * n_lhs);
        const mhg_view vo{&a, out_origin, rows, cols}, vl{&b, lhs_origin, rows, inner},
            vr{&c, rhs_origin, inner, cols};
        const Checked k = check_problem(vo, vl, vr, false, layout_guarded(flags));
        put_counters(counters_of(vo, vl, vr, k, flags), ctr);
    });
}

mhg_status mhg_mm(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, mhg_counters* ctr,
                  void* stream) {
    return mhg_mm_ex(out, lhs, rhs, op, 0u, ctr, stream);
}

mhg_status mhg_mm_ex(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, uint32_t flags,
                     mhg_counters* ctr, void* stream) {
    return guarded([&] {
        if (op != MHG_OP_ADD && op != MHG_OP_SUB && op != MHG_OP_SET)
            fail(MHG_ERR_INVALID_ARGUMENT, "mm: unknown op");
        check_flags(flags);
        const Checked c = check_problem(out, lhs, rhs, (flags & MHG_ALLOW_ALIAS) != 0, layout_guarded(flags));
        const mhg::Counters k = counters_of(out, lhs, rhs, c, flags);
        put_counters(k, ctr);
        if (out.rows == 0 || out.cols == 0) return;
        if (lhs.cols == 0) {
            // empty inner dimension: += / -= leave the view alone (multiply.hpp:303);
            // SET writes zeros, i.e. the product of empty factors
            if (op != MHG_OP_SET) return;
        }
        require_device();
        require_resident({out.mat, lhs.mat, rhs.mat});
        refuse_capture(stream, "mhg_mm");
        const mhg::GemmGeometry g = mhg::gemm_geometry(out.mat->q, c.ro.rows, c.rl.cols, c.ro.cols);
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lock(ws.mu);
        uint8_t* base = ws.acquire(buffer_bytes(c, g), stream);
        const Buffers b = carve(base, c, g);
        launch_offsets_all(b, c, out, lhs, rhs, stream);
        if (lhs.cols == 0)  // SET with k == 0: the product of empty factors is zero
            cuda_check(mhg::launch_fill_view(out.mat->cells, b.out_row, b.out_col, c.ro.rows,
                                             c.ro.cols, 0u, stream),
                       "fill view");
        else
            launch_multiply(b, out, lhs, rhs, c, g, op, stream);
        ws.release(stream);
    });
}

// ------------------------------------------------------------------- plans
mhg_status mhg_plan_create(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, mhg_plan* plan) {
    return mhg_plan_create_ex(out, lhs, rhs, op, 0u, plan);
}

mhg_status mhg_plan_create_ex(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, uint32_t flags,
                              mhg_plan* plan) {
    return guarded([&] {
        if (!plan) fail(MHG_ERR_INVALID_ARGUMENT, "plan_create: null out");
        if (op != MHG_OP_ADD && op != MHG_OP_SUB && op != MHG_OP_SET)
            fail(MHG_ERR_INVALID_ARGUMENT, "plan_create: unknown op");
        check_flags(flags);
        const Checked c = check_problem(out, lhs, rhs, (flags & MHG_ALLOW_ALIAS) != 0, layout_guarded(flags));
        auto* p = new mhg_plan_s();
        p->out = out;
        p->lhs = lhs;
        p->rhs = rhs;
        p->op = op;
        p->chk = c;
        p->ctr = counters_of(out, lhs, rhs, c, flags);
        p->empty = out.rows == 0 || out.cols == 0 || lhs.cols == 0;
        if (p->empty && op == MHG_OP_SET && out.rows && out.cols) {
            delete p;
            fail(MHG_ERR_UNSUPPORTED, "plan: SET with an empty inner dimension (use mhg_mm)");
        }
        if (!p->empty) {
            try {
                require_device();
                require_resident({out.mat, lhs.mat, rhs.mat});
                p->geo = mhg::gemm_geometry(out.mat->q, c.ro.rows, c.rl.cols, c.ro.cols);
                p->mem_bytes = buffer_bytes(c, p->geo);
                cuda_check(cudaMalloc(&p->mem, p->mem_bytes), "plan workspace");
                p->buf = carve(p->mem, c, p->geo);
                launch_offsets_all(p->buf, c, out, lhs, rhs, nullptr);
                cuda_check(cudaStreamSynchronize(nullptr), "plan offsets");
            } catch (...) {
                if (p->mem) cudaFree(p->mem);
                delete p;
                throw;
            }
        }
        *plan = p;
    });
}

// Split execution (multi-GPU panel exchange, paper_1705_04807_b200/dist.py): the owner
// of a segment's operand packs it into the plan's workspace, the packed bytes are
// broadcast to the ranks whose plans have the same geometry, each runs the GEMM.
mhg_status mhg_plan_pack(mhg_plan p, int which, void* stream) {
    return guarded([&] {
        if (!p || (which != 0 && which != 1)) fail(MHG_ERR_INVALID_ARGUMENT, "plan_pack: bad args");
        if (p->empty) return;
        launch_pack_operand(p->buf, p->out, which == 0 ? p->lhs : p->rhs, p->chk, p->geo, p->op, which,
                            stream);
    });
}

mhg_status mhg_plan_pack_buffer(mhg_plan p, int which, void** ptr, uint64_t* bytes) {
    return guarded([&] {
        if (!p || !ptr || !bytes || (which != 0 && which != 1))
            fail(MHG_ERR_INVALID_ARGUMENT, "plan_pack_buffer: bad args");
        *ptr = p->empty ? nullptr : (which == 0 ? (void*)p->buf.apack : (void*)p->buf.bpack);
        *bytes = p->empty ? 0 : (which == 0 ? p->geo.apack_bytes : p->geo.bpack_bytes);
    });
}

mhg_status mhg_plan_gemm(mhg_plan p, void* stream) {
    return guarded([&] {
        if (!p) fail(MHG_ERR_INVALID_ARGUMENT, "plan_gemm: null plan");
        if (p->empty) return;
        if (p->chk.rl.cols == 0) fail(MHG_ERR_INVALID_ARGUMENT, "plan_gemm: empty inner dimension");
        cudaEvent_t b = nullptr, e = nullptr;
        if (p->profiling) {
            if (p->ev_used + 2 > p->ev.size()) {
                const size_t grow = p->ev.size() ? p->ev.size() : 64;
                for (size_t i = 0; i < grow; ++i) {
                    cudaEvent_t ev;
                    cuda_check(cudaEventCreate(&ev), "event");
                    p->ev.push_back(ev);
                }
            }
            b = p->ev[p->ev_used];
            e = p->ev[p->ev_used + 1];
            p->ev_used += 2;
        }
        launch_gemm_stage(p->buf, p->out, p->chk, p->geo, p->op, stream, b, e);
    });
}

mhg_status mhg_plan_run(mhg_plan p, void* stream) {
    return guarded([&] {
        if (!p) fail(MHG_ERR_INVALID_ARGUMENT, "plan_run: null plan");
        if (p->empty) return;
        if (p->profiling) {
            if (p->ev_used + 2 > p->ev.size()) {
                const size_t grow = p->ev.size() ? p->ev.size() : 64;
                for (size_t i = 0; i < grow; ++i) {
                    cudaEvent_t e;
                    cuda_check(cudaEventCreate(&e), "event");
                    p->ev.push_back(e);
                }
            }
            cudaEvent_t b = p->ev[p->ev_used], e = p->ev[p->ev_used + 1];
            p->ev_used += 2;
            cudaStreamCaptureStatus pst = cudaStreamCaptureStatusNone;
            cuda_check(cudaStreamIsCapturing((cudaStream_t)stream, &pst), "capture query");
            if (pst != cudaStreamCaptureStatusNone) {
                launch_multiply(p->buf, p->out, p->lhs, p->rhs, p->chk, p->geo, p->op, stream, b, e);
                return;
            }
            if (!p->pexec) {
                for (auto& ev : p->pev) cuda_check(cudaEventCreate(&ev), "event");
                p->pgraph = capture_graph([&](cudaStream_t cap) {
                    launch_multiply(p->buf, p->out, p->lhs, p->rhs, p->chk, p->geo, p->op, cap, p->pev[0],
                                    p->pev[1]);
                });
                size_t nn = 0;
                cuda_check(cudaGraphGetNodes(p->pgraph, nullptr, &nn), "graph nodes");
                std::vector<cudaGraphNode_t> nodes(nn);
                cuda_check(cudaGraphGetNodes(p->pgraph, nodes.data(), &nn), "graph nodes");
                for (cudaGraphNode_t nd : nodes) {
                    cudaGraphNodeType ty;
                    cuda_check(cudaGraphNodeGetType(nd, &ty), "node type");
                    if (ty != cudaGraphNodeTypeEventRecord) continue;
                    cudaEvent_t ev = nullptr;
                    cuda_check(cudaGraphEventRecordNodeGetEvent(nd, &ev), "event node");
                    for (int k = 0; k < 2; ++k)
                        if (ev == p->pev[k]) p->pnode[k] = nd;
                }
                if (!p->pnode[0] || !p->pnode[1]) fail(MHG_ERR_DEVICE, "profiling graph: event nodes not found");
                cuda_check(cudaGraphInstantiate(&p->pexec, p->pgraph, 0), "graph instantiate");
            }
            cuda_check(cudaGraphExecEventRecordNodeSetEvent(p->pexec, p->pnode[0], b), "set event");
            cuda_check(cudaGraphExecEventRecordNodeSetEvent(p->pexec, p->pnode[1], e), "set event");
            cuda_check(cudaGraphLaunch(p->pexec, (cudaStream_t)stream), "graph launch");
            return;
        }
        cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
        cuda_check(cudaStreamIsCapturing((cudaStream_t)stream, &cap_st), "capture query");
        if (cap_st != cudaStreamCaptureStatusNone) {
            // the caller is capturing its own graph: enqueue the kernels themselves, so they
            // become nodes of that graph
            launch_multiply(p->buf, p->out, p->lhs, p->rhs, p->chk, p->geo, p->op, stream);
            return;
        }
        if (!p->exec) {
            // capture pack(lhs + rhs), gemm once; replay as one graph launch (the kernels'
            // one-time attributes were set outside capture by require_device)
            cudaStream_t cap;
            cuda_check(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
            cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "capture");
            try {
                launch_multiply(p->buf, p->out, p->lhs, p->rhs, p->chk, p->geo, p->op, cap);
            } catch (...) {
                cudaGraph_t g = nullptr;
                cudaStreamEndCapture(cap, &g);
                if (g) cudaGraphDestroy(g);
                cudaStreamDestroy(cap);
                throw;
            }
            cuda_check(cudaStreamEndCapture(cap, &p->graph), "end capture");
            cudaStreamDestroy(cap);
            cuda_check(cudaGraphInstantiate(&p->exec, p->graph, 0), "graph instantiate");
        }
        cuda_check(cudaGraphLaunch(p->exec, (cudaStream_t)stream), "graph launch");
    });
}

// Peer memory for the copy-engine panel exchange (paper_1705_04807_b200/dist.py,
// rank_update_p2p): an owner exports the allocation holding a plan's packed operand,
// the ranks of its row / column group map it once and pull the packed bytes with
// cudaMemcpyAsync, which runs on the copy engines over NVLink and leaves every SM
// to the persistent GEMM (an NCCL broadcast kernel would take SMs from it).
static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(mhg_ipc_handle), "IPC handle size");

mhg_status mhg_ipc_export(const void* ptr, mhg_ipc_handle* handle, uint64_t* offset) {
    return guarded([&] {
        if (!ptr || !handle || !offset) fail(MHG_ERR_INVALID_ARGUMENT, "ipc_export: bad args");
        using Range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static Range range = nullptr;
        if (!range) {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            cuda_check(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q),
                       "cuMemGetAddressRange lookup");
            if (!fn || q != cudaDriverEntryPointSuccess)
                fail(MHG_ERR_DEVICE, "cuMemGetAddressRange unavailable");
            range = reinterpret_cast<Range>(fn);
        }
        CUdeviceptr base = 0;
        size_t size = 0;
        if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
            fail(MHG_ERR_INVALID_ARGUMENT, "ipc_export: not a device allocation");
        cudaIpcMemHandle_t h;
        cuda_check(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle");
        std::memcpy(handle->bytes, &h, sizeof h);
        *offset = (uint64_t)((CUdeviceptr)ptr - base);
    });
}

mhg_status mhg_ipc_open(const mhg_ipc_handle* handle, void** base) {
    return guarded([&] {
        if (!handle || !base) fail(MHG_ERR_INVALID_ARGUMENT, "ipc_open: bad args");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle->bytes, sizeof h);
        cuda_check(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
    });
}

mhg_status mhg_ipc_close(void* base) {
    return guarded([&] {
        if (!base) fail(MHG_ERR_INVALID_ARGUMENT, "ipc_close: null");
        cuda_check(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
    });
}

mhg_status mhg_copy_async(void* dst, const void* src, uint64_t bytes, void* stream) {
    return guarded([&] {
        if ((!dst || !src) && bytes) fail(MHG_ERR_INVALID_ARGUMENT, "copy_async: null pointer");
        if (bytes)
            cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream),
                       "copy_async");
    });
}

// Freivalds verification of a finished multiply (the device analogue of the
// reference's cross-check, bench.hpp:186-193): C_new r == C_old r op A (B r) (mod q)
// for `rounds` random vectors r.  A wrong result passes one round with probability
// <= 1/q.  Synchronous; scratch memory is allocated and freed per call.
mhg_status mhg_verify(mhg_view out_new, mhg_view out_old, mhg_view lhs, mhg_view rhs, mhg_op op,
                      uint32_t rounds, uint64_t seed, int* ok, void* stream) {
    return guarded([&] {
        if (!ok) fail(MHG_ERR_INVALID_ARGUMENT, "verify: null output");
        if (op != MHG_OP_ADD && op != MHG_OP_SUB && op != MHG_OP_SET)
            fail(MHG_ERR_INVALID_ARGUMENT, "verify: unknown op");
        if (rounds == 0) fail(MHG_ERR_INVALID_ARGUMENT, "verify: rounds must be positive");
        const Checked c = check_problem(out_new, lhs, rhs, true, false);
        const mhg::Rect ro = check_view(out_old);
        if (out_old.rows != out_new.rows || out_old.cols != out_new.cols)
            fail(MHG_ERR_LOGIC, "verify: old and new output views differ in shape");
        if (out_old.mat->q != out_new.mat->q) fail(MHG_ERR_LOGIC, "verify: old output uses another modulus");
        *ok = 1;
        const uint64_t r = c.ro.rows, k = c.rl.cols, cc = c.ro.cols;
        if (r == 0 || cc == 0) return;
        require_device();
        require_resident({out_new.mat, out_old.mat, lhs.mat, rhs.mat});
        const uint32_t q = out_new.mat->q;
        cudaStream_t s = (cudaStream_t)stream;
        // tables: new rows/cols, old rows/cols, lhs rows/cols, rhs rows/cols; vectors
        const uint64_t tab = 8 * (2 * r + 2 * cc + r + k + k + cc);
        const uint64_t vec = 4 * (cc + k + 3 * r) + 16;
        uint8_t* mem = nullptr;
        cuda_check(cudaMalloc(&mem, tab + vec + 64), "verify scratch");
        struct Free {
            uint8_t* p;
            ~Free() { cudaFree(p); }
        } guard{mem};
        uint64_t* t = (uint64_t*)mem;
        uint64_t *n_row = t, *n_col = n_row + r, *o_row = n_col + cc, *o_col = o_row + r, *l_row = o_col + cc,
                 *l_col = l_row + r, *r_row = l_col + k, *r_col = r_row + k;
        uint32_t* v = (uint32_t*)(r_col + cc);
        uint32_t *x = v, *y = x + cc, *z = y + k, *wn = z + r, *wo = wn + r;
        int* bad = (int*)(wo + r + 1);
        auto offs = [&](uint64_t* dst, uint64_t start, uint64_t count, uint64_t tside, int is_row) {
            cuda_check(mhg::launch_offsets(dst, start, count, mhg::tile_geom(tside), is_row, s), "verify offsets");
        };
        offs(n_row, c.ro.i, r, out_new.mat->t, 1);
        offs(n_col, c.ro.j, cc, out_new.mat->t, 0);
        offs(o_row, ro.i, r, out_old.mat->t, 1);
        offs(o_col, ro.j, cc, out_old.mat->t, 0);
        offs(l_row, c.rl.i, r, lhs.mat->t, 1);
        offs(l_col, c.rl.j, k, lhs.mat->t, 0);
        offs(r_row, c.rr.i, k, rhs.mat->t, 1);
        offs(r_col, c.rr.j, cc, rhs.mat->t, 0);
        cuda_check(cudaMemsetAsync(bad, 0, sizeof(int), s), "verify flag");
        const int sms = device_info().sms;
        const int mode = op == MHG_OP_ADD ? 0 : (op == MHG_OP_SUB ? 1 : 2);
        for (uint32_t round = 0; round < rounds; ++round) {
            cuda_check(mhg::launch_random_vec(x, cc, seed + 0x9E3779B97F4A7C15ull * (round + 1), q, s), "verify r");
            if (k) {
                cuda_check(mhg::launch_matvec(rhs.mat->cells, r_row, r_col, k, cc, x, y, q, sms, s), "verify Br");
                cuda_check(mhg::launch_matvec(lhs.mat->cells, l_row, l_col, r, k, y, z, q, sms, s), "verify ABr");
            } else {
                cuda_check(cudaMemsetAsync(z, 0, 4 * r, s), "verify zero");  // empty inner dimension
            }
            cuda_check(mhg::launch_matvec(out_new.mat->cells, n_row, n_col, r, cc, x, wn, q, sms, s), "verify Cr");
            if (mode != 2)
                cuda_check(mhg::launch_matvec(out_old.mat->cells, o_row, o_col, r, cc, x, wo, q, sms, s),
                           "verify C0r");
            cuda_check(mhg::launch_freivalds_cmp(wn, wo, z, r, q, mode, bad, s), "verify compare");
        }
        int h = 0;
        cuda_check(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "verify flag");
        cuda_check(cudaStreamSynchronize(s), "verify sync");
        *ok = h ? 0 : 1;
    });
}

// ------------------------------------------------------------ seeded inputs
// mh::Rng (bench.hpp:44-52): mt19937_64(seed) with below(k) = (next * k) >> 64.  The
// benchmark fills containers from it in flat Morton order (gen_problem, :101-103), so
// both arms of bench.py multiply the same residues.
struct mhg_rng_s {
    std::mt19937_64 eng;
};

mhg_status mhg_rng_create(uint64_t seed, mhg_rng* out) {
    return guarded([&] {
        if (!out) fail(MHG_ERR_INVALID_ARGUMENT, "rng_create: null out");
        *out = new mhg_rng_s{std::mt19937_64(seed)};
    });
}

mhg_status mhg_rng_below(mhg_rng g, uint64_t k, uint32_t* dst, uint64_t count) {
    return guarded([&] {
        if (!g || (!dst && count)) fail(MHG_ERR_INVALID_ARGUMENT, "rng_below: null pointer");
        if (k == 0 || k > (uint64_t(1) << 32)) fail(MHG_ERR_INVALID_ARGUMENT, "rng_below: k must be in [1, 2^32]");
        for (uint64_t i = 0; i < count; ++i)
            dst[i] = (uint32_t)(((unsigned __int128)g->eng() * k) >> 64);
    });
}

mhg_status mhg_rng_destroy(mhg_rng g) {
    return guarded([&] { delete g; });
}

mhg_status mhg_plan_counters(mhg_plan p, mhg_counters* ctr) {
    return guarded([&] {
        if (!p) fail(MHG_ERR_INVALID_ARGUMENT, "plan_counters: null plan");
        put_counters(p->ctr, ctr);
    });
}

mhg_status mhg_plan_info(mhg_plan p, uint64_t* launches, uint64_t* tiles, uint32_t* limbs,
                         uint32_t* k_chunks, uint64_t* workspace_bytes) {
    return guarded([&] {
        if (!p) fail(MHG_ERR_INVALID_ARGUMENT, "plan_info: null plan");
        if (launches) *launches = p->empty ? 0 : 2;
        if (tiles) *tiles = (uint64_t)p->geo.Mt * p->geo.Nt;
        if (limbs) *limbs = p->geo.L;
        if (k_chunks) *k_chunks = p->geo.chunks;
        if (workspace_bytes) *workspace_bytes = p->mem_bytes;
    });
}

mhg_status mhg_plan_variant(mhg_plan p, int* unsigned_digits, int* cta_group) {
    return guarded([&] {
        if (!p) fail(MHG_ERR_INVALID_ARGUMENT, "plan_variant: null plan");
        if (unsigned_digits) *unsigned_digits = p->empty ? 0 : (p->geo.udig ? 1 : 0);
        if (cta_group) *cta_group = p->empty ? 0 : (p->geo.pair ? 2 : 1);
    });
}

mhg_status mhg_plan_time_gemm(mhg_plan p, int iters, void* stream, float* ms) {
    return guarded([&] {
        if (!p || iters < 1 || !ms) fail(MHG_ERR_INVALID_ARGUMENT, "plan_time_gemm: bad args");
        if (p->empty) {
            *ms = 0.f;
            return;
        }
        // GEMM alone on the plan's packed operands (as left by the last run);
        // repeated ADD/SUB keep `out` a valid residue container.
        mhg::GemmParams prm = gemm_params(p->buf, p->out, p->chk, p->geo, p->op);
        const TensorMaps tm = tensor_maps(p->buf, p->geo);
        cudaEvent_t a, b;
        cuda_check(cudaEventCreate(&a), "event");
        cuda_check(cudaEventCreate(&b), "event");
        cuda_check(cudaEventRecord(a, (cudaStream_t)stream), "event");
        for (int i = 0; i < iters; ++i)
            launch_gemm_any(prm, p->geo, tm, stream);
        cuda_check(cudaEventRecord(b, (cudaStream_t)stream), "event");
        cuda_check(cudaEventSynchronize(b), "event sync");
        float t = 0.f;
        cudaEventElapsedTime(&t, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *ms = t / (float)iters;
    });
}

mhg_status mhg_plan_set_profiling(mhg_plan p, int enable) {
    return guarded([&] {
        if (!p) fail(MHG_ERR_INVALID_ARGUMENT, "plan_set_profiling: null plan");
        p->profiling = enable != 0;
        p->ev_used = 0;
    });
}

mhg_status mhg_plan_gemm_time(mhg_plan p, float* total_ms, uint64_t* launches) {
    return guarded([&] {
        if (!p || !total_ms) fail(MHG_ERR_INVALID_ARGUMENT, "plan_gemm_time: bad args");
        float sum = 0.f;
        if (p->ev_used) cuda_check(cudaEventSynchronize(p->ev[p->ev_used - 1]), "event sync");
        for (size_t i = 0; i + 1 < p->ev_used; i += 2) {
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]), "elapsed");
            sum += ms;
        }
        *total_ms = sum;
        if (launches) *launches = p->ev_used / 2;
        p->ev_used = 0;
    });
}

mhg_status mhg_plan_destroy(mhg_plan p) {
    return guarded([&] {
        if (!p) return;
        for (cudaEvent_t e : p->ev) cudaEventDestroy(e);
        if (p->pexec) cudaGraphExecDestroy(p->pexec);
        if (p->pgraph) cudaGraphDestroy(p->pgraph);
        for (cudaEvent_t e : p->pev)
            if (e) cudaEventDestroy(e);
        if (p->exec) cudaGraphExecDestroy(p->exec);
        if (p->graph) cudaGraphDestroy(p->graph);
        if (p->mem) cudaFree(p->mem);
        delete p;
    });
}

// ------------------------------------------------------------ plan sequences
mhg_status mhg_sweep_create(const mhg_plan* plans, uint32_t count, mhg_sweep* sweep) {
    return guarded([&] {
        if (!sweep || (!plans && count)) fail(MHG_ERR_INVALID_ARGUMENT, "sweep_create: null pointer");
        if (count == 0) fail(MHG_ERR_INVALID_ARGUMENT, "sweep_create: no plans");
        for (uint32_t i = 0; i < count; ++i) {
            if (!plans[i]) fail(MHG_ERR_INVALID_ARGUMENT, "sweep_create: null plan");
            if (plans[i]->empty) fail(MHG_ERR_UNSUPPORTED, "sweep_create: empty plan in the sequence");
            if (plans[i]->profiling) fail(MHG_ERR_UNSUPPORTED, "sweep_create: plan in profiling mode");
        }
        require_device();
        auto sw = std::unique_ptr<mhg_sweep_s>(new mhg_sweep_s());
        sw->steps = count;
        for (uint32_t i = 0; i < count; ++i) sw->macs += plans[i]->ctr.scalar_macs;
        sw->graph = capture_graph([&](cudaStream_t cap) {
            for (uint32_t i = 0; i < count; ++i) {
                const mhg_plan p = plans[i];
                launch_multiply(p->buf, p->out, p->lhs, p->rhs, p->chk, p->geo, p->op, cap);
            }
        });
        const cudaError_t e = cudaGraphInstantiate(&sw->exec, sw->graph, 0);
        if (e != cudaSuccess) {
            cudaGraphDestroy(sw->graph);
            cuda_check(e, "sweep graph instantiate");
        }
        *sweep = sw.release();
    });
}

mhg_status mhg_sweep_run(mhg_sweep sw, void* stream) {
    return guarded([&] {
        if (!sw) fail(MHG_ERR_INVALID_ARGUMENT, "sweep_run: null sweep");
        cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
        cuda_check(cudaStreamIsCapturing((cudaStream_t)stream, &st), "capture query");
        if (st != cudaStreamCaptureStatusNone)
            fail(MHG_ERR_UNSUPPORTED, "sweep_run: the stream is capturing (run the plans themselves)");
        cuda_check(cudaGraphLaunch(sw->exec, (cudaStream_t)stream), "sweep graph launch");
    });
}

mhg_status mhg_sweep_macs(mhg_sweep sw, uint64_t* macs) {
    return guarded([&] {
        if (!sw || !macs) fail(MHG_ERR_INVALID_ARGUMENT, "sweep_macs: null pointer");
        *macs = sw->macs;
    });
}

mhg_status mhg_sweep_destroy(mhg_sweep sw) {
    return guarded([&] {
        if (!sw) return;
        if (sw->exec) cudaGraphExecDestroy(sw->exec);
        if (sw->graph) cudaGraphDestroy(sw->graph);
        delete sw;
    });
}

// ------------------------------------------------------- multi-GPU partition
namespace {
void dist_fail(int e, const char* what) {
    if (e == 1) fail(MHG_ERR_INVALID_ARGUMENT, std::string(what) + ": rank count must be a power of two");
    if (e == 2) fail(MHG_ERR_OUT_OF_RANGE, std::string(what) + ": rank or segment index out of range");
    if (e == 3) fail(MHG_ERR_INVALID_ARGUMENT, std::string(what) + ": fewer tiles than ranks");
}
}  // namespace

mhg_status mhg_dist_block(uint32_t P, uint32_t rank, uint64_t n, uint64_t t, mhg_dist_block_t* block) {
    mhg_status s = mhg_layout_check(n, t);
    if (s) return s;
    return guarded([&] {
        if (!block) fail(MHG_ERR_INVALID_ARGUMENT, "dist_block: null output");
        mhg::DistBlock b{};
        dist_fail(mhg::dist_block(P, rank, n, t, b), "dist_block");
        *block = mhg_dist_block_t{b.rank, b.i0, b.j0, b.rows, b.cols, b.row_band, b.col_band};
    });
}

mhg_status mhg_dist_slice(uint32_t P, uint32_t rank, uint64_t n, uint64_t* begin, uint64_t* end) {
    return guarded([&] {
        if (!begin || !end) fail(MHG_ERR_INVALID_ARGUMENT, "dist_slice: null output");
        if (P == 0 || (P & (P - 1))) dist_fail(1, "dist_slice");
        if (rank >= P) dist_fail(2, "dist_slice");
        const uint64_t per = n * n / P;
        *begin = rank * per;
        *end = (rank + 1) * per;
    });
}

mhg_status mhg_dist_segment_count(uint32_t P, uint32_t* count) {
    return guarded([&] {
        if (!count) fail(MHG_ERR_INVALID_ARGUMENT, "dist_segment_count: null output");
        const uint32_t c = mhg::dist_segment_count(P);
        if (!c) dist_fail(1, "dist_segment_count");
        *count = c;
    });
}

mhg_status mhg_dist_segment(uint32_t P, uint32_t rank, uint64_t n, uint64_t t, uint32_t index,
                            mhg_dist_segment_t* segment) {
    mhg_status s = mhg_layout_check(n, t);
    if (s) return s;
    return guarded([&] {
        if (!segment) fail(MHG_ERR_INVALID_ARGUMENT, "dist_segment: null output");
        mhg::DistSegment g{};
        dist_fail(mhg::dist_segment(P, rank, n, t, index, g), "dist_segment");
        *segment = mhg_dist_segment_t{g.index, g.k0, g.k1, g.a_owner, g.a_begin, g.a_end,
                                      g.b_owner, g.b_begin, g.b_end};
    });
}

mhg_status mhg_dist_plan_create(mhg_matrix out, mhg_matrix lhs, mhg_matrix rhs, mhg_op op, uint32_t P,
                                uint32_t rank, uint32_t index, mhg_plan* plan) {
    mhg::DistBlock b{};
    mhg::DistSegment g{};
    mhg_status s = guarded([&] {
        if (!out || !lhs || !rhs) fail(MHG_ERR_INVALID_ARGUMENT, "dist_plan_create: null container");
        if (!plan) fail(MHG_ERR_INVALID_ARGUMENT, "dist_plan_create: null out");
        dist_fail(mhg::dist_block(P, rank, out->n, out->t, b), "dist_plan_create");
        dist_fail(mhg::dist_segment(P, rank, out->n, out->t, index, g), "dist_plan_create");
    });
    if (s) return s;
    const uint64_t t = out->t;
    const mhg_view vo{out, mhg::encode(t, b.i0, b.j0), b.rows, b.cols};
    const mhg_view vl{lhs, mhg::encode(t, b.i0, g.k0), b.rows, g.k1 - g.k0};
    const mhg_view vr{rhs, mhg::encode(t, g.k0, b.j0), g.k1 - g.k0, b.cols};
    return mhg_plan_create(vo, vl, vr, (op == MHG_OP_SET && index > 0) ? MHG_OP_ADD : op, plan);
}

}  // extern "C"

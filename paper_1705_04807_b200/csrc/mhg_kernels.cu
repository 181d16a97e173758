// mhg_kernels.cu -- sm_100a kernels of the Morton-hybrid GF(p) MM path.
//
//   K0 k_offsets   Morton offset tables: off(i, j) = rowpart(i) + colpart(j)
//                  (dilate(i/t) << 1 and dilate(j/t) occupy disjoint bits, so the
//                  reference's encode, layout.hpp:80-85, splits into two tables).
//   K1 k_rm_to_mh / k_mh_to_rm
//                  row-major <-> Morton-hybrid permutations (matrix.hpp:44-67),
//                  16-byte coalesced accesses, HBM-bound.
//   K2 k_pack      residue -> L signed int8 limb planes in the exact shared-memory
//                  image of one SWIZZLE_128B K-major UMMA operand stage, so the
//                  GEMM producer moves each stage with ONE cp.async.bulk.
//   K3 k_gemm      persistent warp-specialised tcgen05 kind::i8 GEMM; TMEM holds
//                  the 2L-1 weight classes of the limb products; the epilogue
//                  folds them mod q and applies out (+)= ... at Morton addresses.
//                  Replaces base_case_mm (multiply.hpp:136-172) + add/mul
//                  (field.hpp:43-55).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "mhg_internal.hpp"

namespace mhg {
namespace {

// ------------------------------------------------------------ index helpers
__device__ __forceinline__ uint64_t dilate32(uint64_t x) {
    if (x <= 0xffffull) {
        // tile grids up to 2^16 per side (every n <= 65536): 32-bit arithmetic
        uint32_t y = (uint32_t)x;
        y = (y | (y << 8)) & 0x00ff00ffu;
        y = (y | (y << 4)) & 0x0f0f0f0fu;
        y = (y | (y << 2)) & 0x33333333u;
        y = (y | (y << 1)) & 0x55555555u;
        return y;
    }
    x &= 0xffffffffull;
    x = (x | (x << 16)) & 0x0000ffff0000ffffull;
    x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
    x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

__device__ __forceinline__ void tdivmod(uint64_t v, const TileGeom& g, uint64_t& q, uint64_t& r) {
    if (g.shift >= 0) {
        q = v >> g.shift;
        r = v & (g.t - 1);
    } else {
        q = v / g.t;
        r = v - q * g.t;
    }
}

__device__ __forceinline__ uint64_t rowpart(uint64_t i, const TileGeom& g) {
    uint64_t b, r;
    tdivmod(i, g, b, r);
    if (g.shift >= 0) return (dilate32(b) << (2 * g.shift + 1)) | (r << g.shift);
    return (dilate32(b) << 1) * g.tt + r * g.t;
}

__device__ __forceinline__ uint64_t colpart(uint64_t j, const TileGeom& g) {
    uint64_t b, r;
    tdivmod(j, g, b, r);
    if (g.shift >= 0) return (dilate32(b) << (2 * g.shift)) | r;
    return dilate32(b) * g.tt + r;
}

// ------------------------------------------------------------------- K0
__global__ void k_offsets(uint64_t* __restrict__ dst, uint64_t start, uint64_t count, TileGeom g,
                          int is_row) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < count;
         x += (uint64_t)gridDim.x * blockDim.x)
        dst[x] = is_row ? rowpart(start + x, g) : colpart(start + x, g);
}

// ------------------------------------------------------------------- K1
// Each thread moves 4 consecutive columns of one row.  With t % 4 == 0 the
// four Morton destinations are contiguous (one tile row), so both sides use
// 16-byte accesses; otherwise it falls back to scalar addressing.
__global__ void k_rm_to_mh(const uint32_t* __restrict__ rm, uint32_t* __restrict__ mh, uint64_t n,
                           TileGeom g, uint32_t q, int* __restrict__ bad) {
    const uint64_t groups = n * n / 4;
    const bool vec = (g.t % 4 == 0) && (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(rm) & 15) == 0);
    int saw_bad = 0;
    if (vec) {
        for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < groups;
             x += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t i = (4 * x) / n, j = (4 * x) % n;
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(rm) + x);
            saw_bad |= (v.x >= q) | (v.y >= q) | (v.z >= q) | (v.w >= q);
            __stcs(reinterpret_cast<uint4*>(mh + rowpart(i, g) + colpart(j, g)), v);
        }
    } else {
        for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n * n;
             x += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t i = x / n, j = x % n;
            const uint32_t v = rm[x];
            saw_bad |= v >= q;
            mh[rowpart(i, g) + colpart(j, g)] = v;
        }
    }
    if (saw_bad) atomicOr(bad, 1);
}

// Inverse of dilate32 on the even bits: compact(dilate32(x)) == x.
__device__ __forceinline__ uint32_t compact32(uint64_t x) {
    if ((x >> 32) == 0) {
        // tile indices below 2^32 (every n <= 65536 tile grid): 32-bit arithmetic
        uint32_t y = (uint32_t)x & 0x55555555u;
        y = (y | (y >> 1)) & 0x33333333u;
        y = (y | (y >> 2)) & 0x0f0f0f0fu;
        y = (y | (y >> 4)) & 0x00ff00ffu;
        y = (y | (y >> 8)) & 0x0000ffffu;
        return y;
    }
    x &= 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
    x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
    x = (x | (x >> 16)) & 0x00000000ffffffffull;
    return (uint32_t)x;
}

// K1 in Morton order (power-of-two t, t % 4 == 0): thread x owns the 16-byte
// group at Morton offset 4x, so the Morton side is one contiguous stream and
// the row-major side moves t*4-byte row runs; no divisions.  to_mh = 1:
// row-major -> Morton (+ residue check), 0: Morton -> row-major.
__global__ void k_conv_z(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, uint64_t n,
                         TileGeom g, uint32_t q, int* __restrict__ bad, int to_mh) {
    const uint64_t groups = n * n / 4;
    const int sh = g.shift;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    int saw_bad = 0;
    // 4 groups per thread per round: all four loads in flight before any store
    for (uint64_t x0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x0 < groups; x0 += 4 * stride) {
        uint64_t r[4];
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t x = x0 + u * stride;
            const uint64_t z = 4 * (x < groups ? x : 0);
            const uint64_t tile = z >> (2 * sh);
            const uint64_t rem = z & (g.tt - 1);
            const uint64_t i = ((uint64_t)compact32(tile >> 1) << sh) + (rem >> sh);
            const uint64_t j = ((uint64_t)compact32(tile) << sh) + (rem & (g.t - 1));
            r[u] = i * n + j;
            v[u] = to_mh ? __ldcs(reinterpret_cast<const uint4*>(src + r[u]))
                         : __ldcs(reinterpret_cast<const uint4*>(src) + (x < groups ? x : 0));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t x = x0 + u * stride;
            if (x >= groups) break;
            if (to_mh) {
                saw_bad |= (v[u].x >= q) | (v[u].y >= q) | (v[u].z >= q) | (v[u].w >= q);
                __stcs(reinterpret_cast<uint4*>(dst) + x, v[u]);
            } else {
                __stcs(reinterpret_cast<uint4*>(dst + r[u]), v[u]);
            }
        }
    }
    if (saw_bad) atomicOr(bad, 1);
}

__global__ void k_mh_to_rm(const uint32_t* __restrict__ mh, uint32_t* __restrict__ rm, uint64_t n,
                           TileGeom g) {
    const uint64_t groups = n * n / 4;
    const bool vec = (g.t % 4 == 0) && (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(rm) & 15) == 0);
    if (vec) {
        // 4 groups per thread per round: all four loads in flight before any store;
        // power-of-two n (power-of-two t) splits the flat index with shifts
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        const int ns = 63 - __clzll((long long)n);
        const bool npow2 = (uint64_t(1) << ns) == n;
        for (uint64_t x0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x0 < groups;
             x0 += 4 * stride) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t x = x0 + u * stride;
                const uint64_t f = 4 * (x < groups ? x : 0);
                const uint64_t i = npow2 ? f >> ns : f / n;
                const uint64_t j = npow2 ? f & (n - 1) : f - i * n;
                v[u] = __ldcs(reinterpret_cast<const uint4*>(mh + rowpart(i, g) + colpart(j, g)));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t x = x0 + u * stride;
                if (x >= groups) break;
                __stcs(reinterpret_cast<uint4*>(rm) + x, v[u]);
            }
        }
    } else {
        for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n * n;
             x += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t i = x / n, j = x % n;
            rm[x] = mh[rowpart(i, g) + colpart(j, g)];
        }
    }
}

// ------------------------------------------------------------------- K2
template <int L>
__device__ __forceinline__ void to_digits(uint32_t v, const DigitParams& dp, int8_t (&d)[L]) {
    if (dp.negate) v = v ? dp.q - v : 0u;
    if (dp.udig) {
#pragma unroll
        for (int s = 0; s < L; ++s) d[s] = (int8_t)(uint8_t)(v >> (8 * s));
        return;
    }
    int32_t x = v > dp.H ? (int32_t)(v - dp.q) : (int32_t)v;
#pragma unroll
    for (int s = 0; s < L - 1; ++s) {
        const int8_t lo = (int8_t)(x & 0xff);
        d[s] = lo;
        x = (x - (int32_t)lo) >> 8;
    }
    d[L - 1] = (int8_t)x;
}

// 4 residues -> 4 digits per limb packed little-endian into one 32-bit word
template <int L>
__device__ __forceinline__ void digits4(const uint32_t (&v)[4], const DigitParams& dp,
                                        uint32_t (&w)[L]) {
#pragma unroll
    for (int s = 0; s < L; ++s) w[s] = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        int8_t d[L];
        to_digits<L>(v[e], dp, d);
#pragma unroll
        for (int s = 0; s < L; ++s) w[s] |= (uint32_t)(uint8_t)d[s] << (8 * e);
    }
}

// Four 16-byte runs of a view: rows ri[a] (view coordinates), columns c0..c0+3,
// through the view's offset tables (L1-resident: neighbouring threads share
// entries).  All six table loads go out together, then the four data loads are
// issued unconditionally -- a dead lane reads cell 0 -- so they are all in
// flight at once (a predicated load is followed by register moves that wait
// for it, which serialised this loop before).  Lanes whose run is not one
// aligned 16-byte run (view edges, t % 4 != 0, runs crossing a tile row) are then
// refilled element by element; cells outside the view read as 0.
__device__ __forceinline__ void load4x4(const uint32_t* __restrict__ src,
                                        const uint64_t* __restrict__ rowoff,
                                        const uint64_t* __restrict__ coloff, bool vecok,
                                        const uint64_t (&ri)[4], uint64_t nrows, uint64_t c0,
                                        uint64_t ncols, uint4 (&v)[4]) {
    const uint64_t clast = ncols - 1;
    const uint64_t ca = __ldg(coloff + (c0 < ncols ? c0 : clast));
    const uint64_t cb = __ldg(coloff + (c0 + 3 < ncols ? c0 + 3 : clast));
    uint64_t rb[4];
    bool ok[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        ok[a] = ri[a] < nrows;
        rb[a] = __ldg(rowoff + (ok[a] ? ri[a] : 0));
    }
    const bool cvec = vecok && c0 + 3 < ncols && cb == ca + 3 && (ca & 3) == 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
        v[a] = __ldcs(reinterpret_cast<const uint4*>(src + ((ok[a] && cvec) ? rb[a] + ca : 0)));
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (ok[a] && cvec) continue;
        auto cell = [&](uint64_t e) -> uint32_t {
            return (ok[a] && c0 + e < ncols) ? src[rb[a] + __ldg(coloff + c0 + e)] : 0u;
        };
        v[a] = make_uint4(cell(0), cell(1), cell(2), cell(3));
    }
}

// Swizzle of the K-major UMMA operand image with BK-byte rows (SWIZZLE_<BK>B):
// the 16-byte chunk c of row r sits at chunk c ^ ((r * BK >> 7) & (BK/16 - 1)).
__host__ __device__ constexpr uint32_t swizzled_chunk(uint32_t row, uint32_t chunk) {
    return chunk ^ (((row * (uint32_t)kBK) >> 7) & (uint32_t)(kBK / 16 - 1));
}

// Destination of the 16-byte chunk holding K bytes [kk, kk+16) of pack row pr,
// limb s, in the [row tile][k tile][L][rows_per_tile][BK B] swizzled image.
template <int L>
__device__ __forceinline__ int8_t* pack_dst(int8_t* dst, uint64_t pr, uint64_t kk, int s,
                                            uint32_t rpt, uint32_t Kt) {
    // rows per tile is a power of two (128 for the lhs, W for the rhs): shift, not divide
    const int rs = __ffs(rpt) - 1;
    const uint64_t tile = pr >> rs;
    const uint32_t rit = (uint32_t)(pr & (rpt - 1));
    const uint64_t kt = kk / kBK;
    const uint32_t ch = (uint32_t)(kk % kBK) >> 4;
    return dst + ((tile * Kt + kt) * L + s) * (uint64_t)rpt * kBK + (uint64_t)rit * kBK +
           (swizzled_chunk(rit, ch) << 4);
}

// lhs: pack rows = view rows, K = view columns (contiguous in the source).
// Block: 32 pack rows x 128 K; thread: 4 rows x 4 consecutive K (one 16-byte load
// per row).  Smem holds the digit bytes [L][32][128 (+16 pad)].
constexpr int kRowsStride = kPackK + 16;

// 8 resident blocks per SM (32 registers): full occupancy keeps 4 x 16 B loads per
// thread x 2048 threads in flight -- 0.91 of measured HBM (profiles/r01_pack.txt)
#ifndef MHG_PACK_MINB
#define MHG_PACK_MINB 8
#endif
template <int L>
__device__ __forceinline__ void pack_rows_block(uint32_t bid, const uint32_t* __restrict__ src,
                                                const uint64_t* __restrict__ rowoff,
                                                const uint64_t* __restrict__ coloff, int vecok,
                                                uint64_t R, uint64_t K, uint32_t rpt, uint32_t Kt,
                                                uint64_t Rpad, int8_t* __restrict__ dst,
                                                const DigitParams& dp, uint8_t* smem) {
    auto& sd = *reinterpret_cast<uint8_t(*)[L][32][kRowsStride]>(smem);
    const uint64_t kpad = (uint64_t)Kt * kBK;
    const uint32_t nkb = (uint32_t)((kpad + kPackK - 1) / kPackK);
    const uint32_t kb = bid % nkb;
    const uint64_t pr0 = (uint64_t)(bid / nkb) * 32;
    const uint64_t k0 = (uint64_t)kb * kPackK;
    const int tk = threadIdx.x & 31, tr = threadIdx.x >> 5;
    uint64_t ri[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) ri[a] = pr0 + 4 * tr + a;
    uint4 v4[4];
    load4x4(src, rowoff, coloff, vecok, ri, R, k0 + 4 * tk, K, v4);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = 4 * tr + a;
        const uint32_t v[4] = {v4[a].x, v4[a].y, v4[a].z, v4[a].w};
        uint32_t w[L];
        digits4<L>(v, dp, w);
#pragma unroll
        for (int s = 0; s < L; ++s) *reinterpret_cast<uint32_t*>(&sd[s][r][4 * tk]) = w[s];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < L; ++e) {
        const int cid = threadIdx.x + 256 * e;  // L x 32 rows x 8 chunks
        const int s = cid >> 8, r = (cid >> 3) & 31, ch = cid & 7;
        const uint64_t pr = pr0 + r;
        if (pr >= Rpad || k0 + 16 * ch >= kpad) continue;
        const uint4 val = *reinterpret_cast<const uint4*>(&sd[s][r][ch * 16]);
        *reinterpret_cast<uint4*>(pack_dst<L>(dst, pr, k0 + 16 * ch, s, rpt, Kt)) = val;
    }
}

template <int L>
__global__ void __launch_bounds__(256, MHG_PACK_MINB) k_pack_rows(const uint32_t* __restrict__ src,
                                                   const uint64_t* __restrict__ rowoff,
                                                   const uint64_t* __restrict__ coloff, int vecok,
                                                   uint64_t R, uint64_t K, uint32_t rpt, uint32_t Kt,
                                                   uint64_t Rpad, int8_t* __restrict__ dst,
                                                   DigitParams dp) {
    __shared__ __align__(16) uint8_t sd[L * 32 * kRowsStride];
    pack_rows_block<L>(blockIdx.x, src, rowoff, coloff, vecok, R, K, rpt, Kt, Rpad, dst, dp, sd);
}

// rhs (transposed to K-major): pack rows = view columns (contiguous in the
// source), K = view rows.  Block: 128 pack rows x 32 K; thread: 4 consecutive
// pack rows (one 16-byte load) x 4 K rows, transposed in registers.
constexpr int kColsStride = 36;  // 32 K bytes + 4 pad

template <int L>
__device__ __forceinline__ void pack_cols_block(uint32_t bid, const uint32_t* __restrict__ src,
                                                const uint64_t* __restrict__ rowoff,
                                                const uint64_t* __restrict__ coloff, int vecok,
                                                uint64_t R, uint64_t K, uint32_t rpt, uint32_t Kt,
                                                uint64_t Rpad, int8_t* __restrict__ dst,
                                                const DigitParams& dp, uint8_t* smem) {
    auto& sd = *reinterpret_cast<uint8_t(*)[L][128][kColsStride]>(smem);
    const uint32_t nkq = Kt * (kBK / 32);         // 32-wide K slices
    const uint32_t kq = bid % nkq;
    const uint64_t pr0 = (uint64_t)(bid / nkq) * 128;
    const uint64_t k0 = (uint64_t)kq * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    uint64_t ki[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) ki[i] = k0 + 4 * ty + i;
    uint4 v4[4];  // [k] x 4 pack rows
    load4x4(src, rowoff, coloff, vecok, ki, K, pr0 + 4 * tx, R, v4);
    const uint32_t v[4][4] = {{v4[0].x, v4[0].y, v4[0].z, v4[0].w},
                              {v4[1].x, v4[1].y, v4[1].z, v4[1].w},
                              {v4[2].x, v4[2].y, v4[2].z, v4[2].w},
                              {v4[3].x, v4[3].y, v4[3].z, v4[3].w}};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t col[4] = {v[0][c], v[1][c], v[2][c], v[3][c]};
        uint32_t w[L];
        digits4<L>(col, dp, w);
#pragma unroll
        for (int s = 0; s < L; ++s) *reinterpret_cast<uint32_t*>(&sd[s][4 * tx + c][4 * ty]) = w[s];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < L; ++e) {
        const int cid = threadIdx.x + 256 * e;  // L x 128 rows x 2 chunks
        const int s = cid >> 8, r = (cid >> 1) & 127, h = cid & 1;
        const uint64_t pr = pr0 + r;
        if (pr >= Rpad) continue;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&sd[s][r][16 * h]);
        *reinterpret_cast<uint4*>(pack_dst<L>(dst, pr, k0 + 16 * h, s, rpt, Kt)) =
            make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int L>
__global__ void __launch_bounds__(256, MHG_PACK_MINB) k_pack_cols(const uint32_t* __restrict__ src,
                                                   const uint64_t* __restrict__ rowoff,
                                                   const uint64_t* __restrict__ coloff, int vecok,
                                                   uint64_t R, uint64_t K, uint32_t rpt, uint32_t Kt,
                                                   uint64_t Rpad, int8_t* __restrict__ dst,
                                                   DigitParams dp) {
    __shared__ __align__(16) uint8_t sd[L * 128 * kColsStride];
    pack_cols_block<L>(blockIdx.x, src, rowoff, coloff, vecok, R, K, rpt, Kt, Rpad, dst, dp, sd);
}

// Both operands of a multiply in ONE launch: blocks [0, nrows) pack the lhs (rows
// kernel body), the rest the rhs (cols body).  Two HBM-bound grids of ~2 waves
// each otherwise pay two ramp-down tails (the second graph branch started ~9 us
// late at cfg3, profiles/r01_pack_fused.txt).
template <int L>
__global__ void __launch_bounds__(256, MHG_PACK_MINB) k_pack_pair(PackArgs a, PackArgs b,
                                                                  uint32_t nrows) {
    constexpr int ROWS_SMEM = L * 32 * kRowsStride, COLS_SMEM = L * 128 * kColsStride;
    __shared__ __align__(16) uint8_t sd[ROWS_SMEM > COLS_SMEM ? ROWS_SMEM : COLS_SMEM];
    // programmatic dependent launch: the GEMM that follows may start its prologue (TMEM
    // allocation, barrier init) while the packs drain; it waits (griddepcontrol.wait) for this
    // grid's completion before touching the operands
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (blockIdx.x < nrows)
        pack_rows_block<L>(blockIdx.x, a.src, a.rowoff, a.coloff, a.vecok, a.R, a.K, a.rpt, a.Kt,
                           a.Rpad, a.dst, a.dp, sd);
    else
        pack_cols_block<L>(blockIdx.x - nrows, b.src, b.rowoff, b.coloff, b.vecok, b.R, b.K, b.rpt,
                              b.Kt, b.Rpad, b.dst, b.dp, sd);
}

// ------------------------------------------------------------------- K3
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Blocking wait with a suspend-time hint (ns): the thread sleeps in the
// barrier until the phase completes instead of re-polling, which keeps the
// single-thread producer / MMA roles off the issue slots their SMSP shares with
// epilogue warps.
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
    if (hint_ns == 0) {
        mbar_wait(bar, parity);
        return;
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(hint_ns)
        : "memory");
}

// Wait-cycle counters of the GEMM roles (MHG_OPT_GEMM_STATS, profiles/gemm_stats*.py) are
// compiled only into diagnostic builds (-DMHG_DIAG=1, profiles/build_variant.sh): in the
// product build diag_clock() is the constant 0, the counters fold away and take no
// registers (they cost ~14 in the epilogue, where the 10-warp CTA is capped at 168).
#ifndef MHG_DIAG
#define MHG_DIAG 0
#endif

__device__ __forceinline__ long long diag_clock() {
#if MHG_DIAG
    return clock64();
#else
    return 0;
#endif
}

// global C_old / C accesses of the coalesced epilogue: streaming (.cs) -- measured
// best against default caching and L1::no_allocate (profiles/r01_epilogue_ab.txt)
__device__ __forceinline__ uint4 c_load(const uint4* a) { return __ldcs(a); }

// 16-byte global -> shared copy through the LSU (cp.async, no registers); src_bytes = 0
// zero-fills the destination
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void c_store(uint4* a, uint4 v) { __stcs(a, v); }

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// named barrier among the 4 epilogue warps (id 1; id 0 is __syncthreads)
template <int N>
__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory"); }

// Bulk copy with an L2 eviction-priority policy (createpolicy result).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, int8 x int8 -> int32
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// K-major operand, SWIZZLE_<BK>B: 8-row x BK-byte atoms, 8*BK bytes apart (SBO).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    static_assert(kBK == 128 || kBK == 64, "swizzle width");
    constexpr uint64_t layout = kBK == 128 ? 2 : 4;  // SWIZZLE_128B / SWIZZLE_64B
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * kBK) >> 4) << 32;     // SBO
    d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
    d |= layout << 61;
    return d;
}

// kind::i8 instruction descriptor: s8 x s8 -> s32, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4)                   // D format S32
           | (1u << 7)                 // A signed
           | (1u << 10)                // B signed
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// clearing these makes both operands unsigned (u8 x u8)
__host__ __device__ constexpr uint32_t idesc_sign_mask() { return (1u << 7) | (1u << 10); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// Two x16 loads and the wait in ONE asm statement: the compiler cannot consume the first
// load's registers (scheduling its arithmetic between the loads) before the second is issued
// and both have landed -- both loads are in flight together.
__device__ __forceinline__ void tmem_ld16x2_wait(uint32_t ta, uint32_t tb, int32_t (&a)[16], int32_t (&b)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%32];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%33];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
          "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]),
          "=r"(a[13]), "=r"(a[14]), "=r"(a[15]),
          "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]),
          "=r"(b[7]), "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]),
          "=r"(b[13]), "=r"(b[14]), "=r"(b[15])
        : "r"(ta), "r"(tb)
        : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, int32_t (&v)[N]) {
    if constexpr (N == 16) tmem_ld16(taddr, v);
    else tmem_ld8(taddr, v);
}

__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// x mod q for |x| < 2^62 (bias = multiple of q >= 2^62 makes it non-negative)
__device__ __forceinline__ uint32_t red_signed(int64_t x, const GemmParams& p) {
    const uint64_t u = (uint64_t)x + p.bias;
    const uint64_t qt = __umul64hi(u, p.mu);
    uint64_t r = u - qt * p.q;
    r = r >= p.q ? r - p.q : r;
    r = r >= p.q ? r - p.q : r;
    return (uint32_t)r;
}

__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, const GemmParams& p) {
    const uint64_t u = (uint64_t)a * b;
    const uint64_t qt = __umul64hi(u, p.mu);
    uint64_t r = u - qt * p.q;
    r = r >= p.q ? r - p.q : r;
    r = r >= p.q ? r - p.q : r;
    return (uint32_t)r;
}

// u mod q for u < 2^32, q <= 2^16: Barrett with m = floor(2^32/q) is off by at
// most one multiple of q.
__device__ __forceinline__ uint32_t red32(uint32_t u, const GemmParams& p) {
    const uint32_t r = __umulhi(u, p.m32) * p.nq + u;  // u - floor(u m32 / 2^32) q
    return umin(r, r + p.nq);  // r < 2q: r - q wraps above r when r < q
}

// Fold the 2L-1 weight classes of one output element to a canonical residue:
// S = sum_c acc_c 256^c (mod q).  L <= 2 (q <= 2^16) stays in 32 bits (class 0
// and class 2L-2 are single-product sums, |a| <= 2^30; every class is within
// 2^31 - 2^17 by the planner's K bound); wider primes fold exactly in int64.
template <int L, int CW>
__device__ __forceinline__ uint32_t fold_classes(const int32_t (&acc)[2 * L - 1][CW], int j,
                                                 const GemmParams& p) {
    if constexpr (L == 1) {
        return red32((uint32_t)acc[0][j] + p.bias32, p);
    } else if constexpr (L == 2) {
        const uint32_t r1 = red32((uint32_t)acc[1][j] + p.bias32, p);
        const uint32_t r2 = red32((uint32_t)acc[2][j] + p.bias32, p);
        const uint32_t u = (uint32_t)acc[0][j] + p.bias32 + (r1 << 8);
        if (p.w16_small) return red32(u + p.w16 * r2, p);
        const uint32_t x = red32(u, p) + red32(p.w16 * r2, p);
        return x >= p.q ? x - p.q : x;
    } else {
        int64_t lo = 0, hi = 0;
#pragma unroll
        for (int k = 0; k < 2 * L - 1; ++k) {
            if (k < 4) lo += (int64_t)acc[k][j] << (8 * k);
            else hi += (int64_t)acc[k][j] << (8 * (k - 4));
        }
        uint32_t r = red_signed(lo, p);
        if (2 * L - 1 > 4) {
            const uint32_t h = mulmod(red_signed(hi, p), p.w32, p);
            r += h;
            r = r >= p.q ? r - p.q : r;
        }
        return r;
    }
}

// Whether accumulation jobs alternate TMEM bases 0 / W so that the epilogue can
// release TMEM before draining the last class group (single-CTA kernel).  Pays
// when the early group is cheap: L = 1 (full double buffering) and L = 2 with
// 2^16 mod q < 256; wider primes keep the fused single-phase drain.
template <int L>
__device__ __forceinline__ bool early_release(const GemmParams& p) {
    return L == 1 || (L == 2 && p.w16_small);
}

// Partial fold over the weight classes [C0, C1): sum_c acc[c - C0] 256^c mod q
// (the epilogue drains a job's classes in two groups, see epilogue_role).
template <int L, int CW, int C0, int C1>
__device__ __forceinline__ uint32_t fold_part(const int32_t (&acc)[C1 - C0][CW], int j,
                                              const GemmParams& p) {
    if constexpr (L <= 2) {
        uint32_t x = 0;
#pragma unroll
        for (int c = C0; c < C1; ++c) {
            const uint32_t r = red32((uint32_t)acc[c - C0][j] + p.bias32, p);
            uint32_t term = r;
            if (c == 1) term = red32(r << 8, p);          // 256 r < 2^24
            if (c == 2) term = red32(p.w16 * r, p);       // (2^16 mod q) r < 2^32
            x += term;
            x = x >= p.q ? x - p.q : x;
        }
        return x;
    } else {
        int64_t lo = 0, hi = 0;
        bool any_hi = false;
#pragma unroll
        for (int c = C0; c < C1; ++c) {
            if (c < 4) lo += (int64_t)acc[c - C0][j] << (8 * c);
            else {
                hi += (int64_t)acc[c - C0][j] << (8 * (c - 4));
                any_hi = true;
            }
        }
        uint32_t r = red_signed(lo, p);
        if (any_hi) {
            const uint32_t h = mulmod(red_signed(hi, p), p.w32, p);
            r += h;
            r = r >= p.q ? r - p.q : r;
        }
        return r;
    }
}

#ifndef MHG_SMR
#define MHG_SMR 1
#endif
#define MHG_SMR_CTL_REGS 56   // warpgroup 0 after setmaxnreg.dec
#define MHG_SMR_EPI_REGS 224  // epilogue warpgroups after setmaxnreg.inc (128*56 + 256*224 <= 64K)
#ifndef MHG_DRAIN_PIPE
#define MHG_DRAIN_PIPE MHG_SMR  // all TMEM loads of a drain group in flight at once (needs the registers)
#endif
#ifndef MHG_XADDR_VOLATILE
#define MHG_XADDR_VOLATILE 1  // transpose-buffer addresses recomputed per use (fewer spills)
#endif
#ifndef MHG_COLD_MID
#define MHG_COLD_MID 2  // C_old requested between the two drain groups: 1 = pass 0, 2 = both passes
#endif
// NARROW: 128 x 64 tiles for 1-2 limb primes (GemmGeometry::narrow), chosen for problems of
// at most half a wave of 128 x 128 tiles: twice the CTAs, each with half the MMA and epilogue
// work of the latency chain that bounds such problems (cfg1: 16 -> 32 CTAs).
template <int L, bool NARROW = false>
struct GemmCfg {
    static_assert(!NARROW || L <= 2, "narrow tiles are the 1-2 limb case");
    static constexpr int W = (L <= 2 && !NARROW) ? 128 : 64;  // output columns per tile
    static constexpr int NB = L * W;                    // UMMA N of the stacked B'
    static constexpr int CLASSES = 2 * L - 1;           // weight classes 256^c
    static constexpr int A_STAGE = L * kBM * kBK;       // bytes
    static constexpr int B_STAGE = NB * kBK;            // bytes
    static constexpr int STAGE = A_STAGE + B_STAGE;
    // two epilogue warps per SMSP, 64 columns each; W = 128 uses the coalesced
    // C path with a 4 KB per-warp transpose buffer, the narrow-tile primes keep
    // row-per-thread C access (see epilogue_role)
    static constexpr bool XPOSE = (W == 128) || NARROW;
    static constexpr int EPI_WARPS = 8;
    // MHG_SMR: warpgroup 0 = producer, MMA issuer and two idle warps, which give registers
    // back (setmaxnreg.dec) so the two epilogue warpgroups run at SMR_EPI_REGS instead of the
    // 168 a 10-warp CTA is capped at (three warps share SMSPs 0 and 1)
    static constexpr int EPI_W0 = MHG_SMR ? 4 : 2;  // first epilogue warp
    static constexpr int XBUF = XPOSE ? EPI_WARPS * (W * 4 / EPI_WARPS >= 64 ? 4096 : 2048) : 0;
    static constexpr int FIXED = 1024 /*align slack*/ + 256 /*barriers*/ + 8 * W /*column offsets*/ + XBUF;
    static constexpr int STAGES_RAW = (232448 - FIXED) / STAGE;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static constexpr int SMEM = FIXED + STAGES * STAGE;
    static_assert(SMEM <= 232448, "227 KB dynamic shared memory limit");
    static constexpr int EPI_THREADS = EPI_WARPS * 32;
    static constexpr int THREADS = 32 * EPI_W0 + EPI_THREADS;  // producer, MMA, (idle,) epilogue
    static_assert(!MHG_SMR || (THREADS == 384 && EPI_WARPS == 8), "setmaxnreg layout: 3 warpgroups");
    static_assert(CLASSES * W <= 512, "TMEM columns");
    static_assert(STAGES >= 2, "pipeline depth");
};

__device__ __forceinline__ void tile_coords(uint32_t tile, uint32_t Mt, uint32_t Nt, uint32_t G,
                                            uint32_t& m, uint32_t& n) {
    // grouped raster: G row tiles iterate over the column tiles together, so the
    // tiles in flight share lhs and rhs panels in L2
    const uint32_t group = G * Nt;
    const uint32_t gid = tile / group;
    const uint32_t first_m = gid * G;
    const uint32_t gm = (Mt - first_m) < G ? (Mt - first_m) : G;
    const uint32_t local = tile - gid * group;
    m = first_m + local % gm;
    n = local / gm;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

__device__ __forceinline__ void tma2d_pair(uint32_t dst, const void* tmap, int c0, int c1,
                                           uint32_t leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(leader_bar)
        : "memory");
}

__device__ __forceinline__ void mma_i8_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}

__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
        "r"(0)
        : "memory");
}

__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
                     taddr),
                 "r"(0)
                 : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_zero(uint32_t taddr) {
    if constexpr (N == 16) tmem_zero16(taddr);
    else tmem_zero8(taddr);
}

__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// K1 through the TMA (power-of-two t, 4 <= t <= 256): the unit is a box of R
// rows x t columns of one tile (R*t*4 <= 16 KB; a whole tile up to t = 64).  Its
// Morton image is one contiguous run (rows of a tile are row-major), its
// row-major image a 2D box of the tensor map `tm` (uint32, n x n).  One thread
// per CTA keeps kConvBufs units in flight: to_mh = 1: 2D tensor load -> smem ->
// (residue check by all threads) -> 1D bulk store; to_mh = 0: 1D bulk load ->
// smem -> 2D tensor store.  No data passes through registers except the check.
constexpr int kConvUnitBytes = 16384;
// 4 units in flight per CTA x 3 CTAs per SM (more independent issuers measured faster
// than fewer, deeper CTAs: profiles/r01_conversion_tma.txt)
#ifndef MHG_CONV_UNITS
#define MHG_CONV_UNITS 4
#endif
#ifndef MHG_CONV_CTAS
#define MHG_CONV_CTAS 3
#endif
constexpr int kConvUnits = MHG_CONV_UNITS, kConvCtasPerSm = MHG_CONV_CTAS;
#ifndef MHG_CONV_DEFER
#define MHG_CONV_DEFER 1  // refill a buffer one unit after its store was issued
#endif

__device__ __forceinline__ void tma2d_load(uint32_t dst, const CUtensorMap* tm, int c0, int c1,
                                           uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma2d_store(const CUtensorMap* tm, int c0, int c1, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int kConvBufs>
__global__ void __launch_bounds__(128) k_conv_tma(const __grid_constant__ CUtensorMap tm,
                                                  uint32_t* __restrict__ mh, uint64_t n, TileGeom g,
                                                  uint32_t R, uint32_t q, int* __restrict__ bad,
                                                  int to_mh) {
    extern __shared__ uint8_t conv_raw[];
    uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(conv_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kConvBufs];
    const uint32_t t = (uint32_t)g.t;
    const uint32_t ubytes = R * t * 4;
    const uint32_t upt = t / R;  // units per tile
    const uint64_t units = n * n / ((uint64_t)R * t);
    const bool issuer = threadIdx.x == 0;
    if (issuer) {
        for (int b = 0; b < kConvBufs; ++b) mbar_init(&full[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // unit u: tile z = u / upt (Z order), rows [ (u % upt) R, +R ) of that tile
    auto coords = [&](uint64_t u, int& c0, int& c1, uint64_t& zoff) {
        const uint64_t z = u / upt;
        const uint32_t part = (uint32_t)(u % upt);
        c0 = (int)((uint64_t)compact32(z) * t);
        c1 = (int)((uint64_t)compact32(z >> 1) * t + part * R);
        zoff = z * g.tt + (uint64_t)part * R * t;
    };
    auto issue_load = [&](uint64_t u, int b) {
        int c0, c1;
        uint64_t zoff;
        coords(u, c0, c1, zoff);
        mbar_expect_tx(&full[b], ubytes);
        if (to_mh) tma2d_load(smem_u32(buf + b * kConvUnitBytes), &tm, c0, c1, &full[b]);
        else bulk_g2s(buf + b * kConvUnitBytes, mh + zoff, ubytes, &full[b]);
    };
    const uint64_t first = blockIdx.x, step = gridDim.x;
    if (issuer) {
        uint64_t u = first;
        for (int b = 0; b < kConvBufs && u < units; ++b, u += step) issue_load(u, b);
    }
    int saw_bad = 0;
    uint32_t k = 0;
    for (uint64_t u = first; u < units; u += step, ++k) {
        const int b = (int)(k % kConvBufs);
        const uint32_t phase = (k / kConvBufs) & 1;
        if (to_mh) {
            mbar_wait(&full[b], phase);
            const uint4* v = reinterpret_cast<const uint4*>(buf + b * kConvUnitBytes);
            for (uint32_t i = threadIdx.x; i < ubytes / 16; i += blockDim.x) {
                const uint4 x = v[i];
                saw_bad |= (x.x >= q) | (x.y >= q) | (x.z >= q) | (x.w >= q);
            }
            __syncthreads();  // every thread is done reading buffer b
        }
        if (issuer) {
            if (!to_mh) mbar_wait(&full[b], phase);
            int c0, c1;
            uint64_t zoff;
            coords(u, c0, c1, zoff);
            const uint32_t src = smem_u32(buf + b * kConvUnitBytes);
            if (to_mh) bulk_s2g(mh + zoff, src, ubytes);
            else tma2d_store(&tm, c0, c1, src);
            bulk_commit();
#if MHG_CONV_DEFER
            // refill the PREVIOUS unit's buffer: its store (every group but the one just
            // committed) has read shared memory by now, so the issuer does not sit out this
            // store's read before it can serve the next landed unit
            if (k > 0) {
                bulk_wait_read1();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                // unit k - 1 + kConvBufs of this CTA (unit j >= kConvBufs is requested in
                // iteration j - kConvBufs + 1, which always runs when unit j exists)
                const uint64_t nu = u + (uint64_t)(kConvBufs - 1) * step;
                if (nu < units) issue_load(nu, (int)((k - 1) % kConvBufs));
            }
#else
            bulk_wait_read0();  // the store has read buffer b
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint64_t nu = u + (uint64_t)kConvBufs * step;
            if (nu < units) issue_load(nu, b);
#endif
        }
    }
    if (issuer) bulk_wait0();
    if (to_mh && __syncthreads_or(saw_bad) && threadIdx.x == 0) atomicOr(bad, 1);
}

// Epilogue role of both GEMM kernels (warps 2 .. 2+EPI_WARPS-1).  Per tile:
// (1) bring the tile's output rows (C_old) into a register copy; (2) per exact
// K-chunk, drain the 2L-1 weight classes from TMEM (tcgen05.ld 32x32b), fold
// them mod q into the copy and release TMEM; (3) store the copy after the
// release, overlapping the next tile's MMAs.  One TMEM lane (= output row) per
// thread; warp w may only access lane quadrant w % 4, and the EPI_WARPS / 4
// warps of a quadrant split the columns.  PAIR (k_gemm2): the tile's row block
// is 2*pm + rank, the upper classes [L, 2L-1) are re-zeroed as they are drained
// (every MMA but the first of a chunk accumulates), and TMEM is released on the
// LEADER's barrier.
//
// XPOSE (k_gemm, W = 128, 8 warps x 64 columns): C_old is loaded and C is
// stored in a coalesced order -- per warp instruction 8 lanes cover one
// 128-byte row run (32 columns), 4 rows at a time -- and moved to / from the
// row-per-thread copy through a 4 KB per-warp shared buffer (32 rows x 8
// 16-byte chunks, chunk index XOR row%8: both orders bank-conflict free), one
// 32-column pass at a time.  Output offsets are computed from the Morton
// geometry (no table loads).  Otherwise (narrow tiles, CTA pair) the row's
// C_old is prefetched into registers at tile start, addressed through smem
// column offsets.
template <int L, int W, int EPI_WARPS, bool PAIR, bool XPOSE = false, int FOLD = 3, int EW0 = 2>
__device__ __forceinline__ void epilogue_role(const GemmParams& p, uint32_t first_tile,
                                              uint32_t tile_stride, uint32_t num_tiles,
                                              uint32_t row_groups, uint32_t rank, uint32_t nchunks,
                                              uint32_t tmem, uint64_t* s_col, uint64_t* tmem_full,
                                              uint64_t* tmem_empty, int warp, int lane,
                                              uint8_t* xbuf = nullptr) {
    constexpr int EPI_THREADS = EPI_WARPS * 32;
    constexpr int WH = W * 4 / EPI_WARPS;  // columns per epilogue warp
    constexpr int CLASSES = 2 * L - 1;
    constexpr int CW = L <= 2 ? 16 : 8;  // TMEM columns per drain step (x8 / x32 measured slower)
    constexpr uint64_t kNoCol = ~uint64_t(0);
    constexpr int EPI_W0 = EW0;  // first epilogue warp (warps 0, 1: producer, MMA issuer)
    const int ew = warp - EPI_W0;
    const int quad = warp & 3;
    const int jb = (ew >> 2) * WH;  // first tile column of this warp
    const int row = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t release_bar =
        PAIR ? mapa_shared(smem_u32(tmem_empty), 0) : smem_u32(tmem_empty);
    uint32_t acc_ph = 0;
    long long epi_wait = 0, epi_busy = 0, epi_ldw = 0;
    // hand the accumulator columns back to the MMA issuer (one arrive per warp)
    auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            if constexpr (PAIR) mbar_arrive_remote(release_bar);
            else mbar_arrive(tmem_empty);
        }
    };
    // L = 2 with w16 = 2^16 mod q < 256.  Base 0: classes {1,2} first --
    // cur += 256 r1 + w16 r2 (unreduced, < 2^25) -- release, then class 0:
    // cur = red(cur + a0 + bias).  Base W: classes {0,1} first -- cur += a0 +
    // bias + 256 r1 (unreduced, < 2^32 - 2^24) -- release, then class 2:
    // cur = red(cur + w16 r2).  Every class sum is within 2^31 - 2^17 (class 0
    // and class 2 within 2^30), so no step wraps 32 bits.
    // Per-element folds of the two class groups (lean L = 2 path), by FOLD level
    // (host-chosen, GemmParams::fold; each level exact for the chunk's K):
    //   3: reduce every class before combining (three reductions per element);
    //   2: with a1 = 256 a1h + a1l (a1l the low byte), 256 a1 == 256 a1l + w16 a1h
    //      (mod q): only a2 is reduced first (two reductions);
    //   1: a0 + 256 a1l + w16 (a1h + a2) itself stays within 2^31 - 2^17 for
    //      short chunks (one reduction).
    auto fold_g1 = [&](int32_t x, int32_t y, uint32_t layout) -> uint32_t {
        // layout 0: x = a1, y = a2; layout 1: x = a0, y = a1
        if constexpr (FOLD <= 2) {
            if (layout == 0) {
                const uint32_t lo = (((uint32_t)x & 0xffu) << 8);
                if constexpr (FOLD == 1) return lo + p.w16 * (uint32_t)((x >> 8) + y);
                return lo + p.w16 * ((uint32_t)(x >> 8) + red32((uint32_t)y + p.bias32, p));
            }
            return (uint32_t)x + (((uint32_t)y & 0xffu) << 8) + p.w16 * (uint32_t)(y >> 8);
        }
        const uint32_t r1 = red32((uint32_t)(layout ? y : x) + p.bias32, p);
        if (layout == 0) {
            const uint32_t r2 = red32((uint32_t)y + p.bias32, p);
            return (r1 << 8) + p.w16 * r2;
        }
        return (uint32_t)x + p.bias32 + (r1 << 8);
    };
    auto fold_g2 = [&](uint32_t c, int32_t z, uint32_t layout) -> uint32_t {
        // layout 0: z = a0; layout 1: z = a2
        if (layout == 0) return red32(c + (uint32_t)z + p.bias32, p);
        if constexpr (FOLD == 1) return red32(c + p.w16 * (uint32_t)z + p.bias32, p);
        const uint32_t r2 = red32((uint32_t)z + p.bias32, p);
        if constexpr (FOLD == 2) return red32(c + p.w16 * r2 + p.bias32, p);
        return red32(c + p.w16 * r2, p);
    };
    auto drain_l2_small = [&](uint32_t tbase, uint32_t n_tile, uint32_t* cur_, uint32_t layout, auto&& after_release) {
        const int lo_cls = layout ? 0 : 1;  // first group: {lo_cls, lo_cls + 1}
        if constexpr (FOLD == 1) {
            // Both layouts in one code path (half the instructions in the I-cache): with
            // T(a1) = 256 (a1 & 255) + w16 (a1 >> 8), group 1 adds T(a1) + cb * b and group 2
            // reduces cur + cz * z, where (b, cb, z, cz) = (a2, w16, a0, 1) for layout 0 and
            // (a0, 1, a2, w16) for layout 1 -- the two formulas of fold_g1 / fold_g2.
            const uint32_t col_b = layout ? 0u : 2u * W, col_z = layout ? 2u * W : 0u;
            const uint32_t cb = layout ? 1u : p.w16, cz = layout ? p.w16 : 1u;
            static_assert(CW == 16, "x16 drain steps");
#if MHG_DRAIN_PIPE
            // every load of the group in flight before the first fold (the epilogue
            // warpgroups have the registers under MHG_SMR); columns past the view are folded
            // too (never stored)
            {
                int32_t a[WH / CW][2][CW];
#pragma unroll
                for (int s = 0; s < WH / CW; ++s) {
                    tmem_ld16(tbase + W + s * CW, a[s][0]);
                    tmem_ld16(tbase + col_b + s * CW, a[s][1]);
                }
                tmem_wait_ld();
#pragma unroll
                for (int s = 0; s < WH / CW; ++s)
#pragma unroll
                    for (int j = 0; j < CW; ++j) {
                        const uint32_t a1 = (uint32_t)a[s][0][j];
                        cur_[s * CW + j] += ((a1 & 0xffu) << 8) + p.w16 * (uint32_t)(a[s][0][j] >> 8) + cb * (uint32_t)a[s][1][j];
                    }
            }
#else
#pragma unroll
            for (int j0 = 0; j0 < WH; j0 += CW) {
                if ((uint64_t)n_tile * W + jb + j0 >= p.cols) continue;  // warp-uniform
                int32_t a[2][CW];
                tmem_ld16x2_wait(tbase + W + j0, tbase + col_b + j0, a[0], a[1]);
#pragma unroll
                for (int j = 0; j < CW; ++j) {
                    const uint32_t a1 = (uint32_t)a[0][j];
                    cur_[j0 + j] += ((a1 & 0xffu) << 8) + p.w16 * (uint32_t)(a[0][j] >> 8) + cb * (uint32_t)a[1][j];
                }
            }
#endif
            release();
            after_release();
#if MHG_DRAIN_PIPE
            {
                int32_t a[WH / CW][CW];
#pragma unroll
                for (int s = 0; s < WH / CW; ++s) tmem_ld16(tbase + col_z + s * CW, a[s]);
                tmem_wait_ld();
#pragma unroll
                for (int s = 0; s < WH / CW; ++s)
#pragma unroll
                    for (int j = 0; j < CW; ++j)
                        cur_[s * CW + j] = red32(cur_[s * CW + j] + cz * (uint32_t)a[s][j] + p.bias32, p);
            }
#else
#pragma unroll
            for (int j0 = 0; j0 < WH; j0 += CW) {
                if ((uint64_t)n_tile * W + jb + j0 >= p.cols) continue;
                int32_t a[1][CW];
                tmem_ld<CW>(tbase + col_z + j0, a[0]);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < CW; ++j) cur_[j0 + j] = red32(cur_[j0 + j] + cz * (uint32_t)a[0][j] + p.bias32, p);
            }
#endif
            return;
        }
#pragma unroll
        for (int j0 = 0; j0 < WH; j0 += CW) {
            if ((uint64_t)n_tile * W + jb + j0 >= p.cols) continue;  // warp-uniform
            int32_t a[2][CW];
            const long long l0 = diag_clock();
            tmem_ld<CW>(tbase + lo_cls * W + j0, a[0]);
            tmem_ld<CW>(tbase + (lo_cls + 1) * W + j0, a[1]);
            tmem_wait_ld();
            epi_ldw += diag_clock() - l0;
#pragma unroll
            for (int j = 0; j < CW; ++j) cur_[j0 + j] += fold_g1(a[0][j], a[1][j], layout);
        }
        release();
        after_release();
#pragma unroll
        for (int j0 = 0; j0 < WH; j0 += CW) {
            if ((uint64_t)n_tile * W + jb + j0 >= p.cols) continue;
            int32_t a[1][CW];
            const long long l0 = diag_clock();
            tmem_ld<CW>(tbase + (layout ? 2 : 0) * W + j0, a[0]);
            tmem_wait_ld();
            epi_ldw += diag_clock() - l0;
#pragma unroll
            for (int j = 0; j < CW; ++j) cur_[j0 + j] = fold_g2(cur_[j0 + j], a[0][j], layout);
        }
    };
    // drain weight classes [C0, C1) of this warp's columns and fold them into cur
    auto drain = [&](auto c0_tag, auto c1_tag, uint32_t tbase, uint32_t n_tile, uint32_t* cur_) {
        constexpr int C0 = decltype(c0_tag)::value, C1 = decltype(c1_tag)::value;
        if constexpr (C1 > C0) {
#pragma unroll
            for (int j0 = 0; j0 < WH; j0 += CW) {
                if ((uint64_t)n_tile * W + jb + j0 >= p.cols) continue;  // warp-uniform
                int32_t acc[C1 - C0][CW];
#pragma unroll
                for (int k = C0; k < C1; ++k) tmem_ld<CW>(tbase + k * W + j0, acc[k - C0]);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < CW; ++j) {
                    uint32_t r;
                    if constexpr (C0 == 0 && C1 == CLASSES) r = fold_classes<L, CW>(acc, j, p);
                    else r = fold_part<L, CW, C0, C1>(acc, j, p);
                    const uint32_t sum = cur_[j0 + j] + r;
                    cur_[j0 + j] = sum >= p.q ? sum - p.q : sum;
                }
            }
        }
    };
    long long epi_pro = 0, epi_tail = 0, epi_issue = 0, epi_land = 0;
    // ---- XPOSE helpers: coalesced order = rows RPI*i + sr (i < NI), 16-byte
    // chunk ch of a PW-column pass h (NH passes)
    constexpr int PW = WH >= 64 ? 32 : 16, CPR = PW / 4, RPI = 32 / CPR, NI = 32 / RPI, NH = WH / PW;
    const int sr = lane / CPR, ch = lane % CPR;
    const uint32_t xb = XPOSE ? smem_u32(xbuf) + ew * (32 * PW * 4) : 0u;
    // chunk swizzle: 8 chunks per row -> c ^ r%8; 4 chunks -> c ^ (r/2)%4 (each
    // 8-lane phase of a 16-byte access hits 8 distinct bank groups in both orders)
    auto xaddr = [&](int r, int c) -> uint32_t {
        const int sw = CPR == 8 ? (r & 7) : ((r >> 1) & 3);
        uint32_t base = xb;
#if MHG_XADDR_VOLATILE
        // recomputed at each use: hoisted out of the tile loop, the per-lane addresses
        // (16+ registers at the 168-register cap) are spilled and reloaded every tile
        asm volatile("" : "+r"(base));
#endif
        return base + r * (PW * 4) + ((c ^ sw) << 4);
    };
    // container offset of output row m*128 + r (kNoCol past the view)
    auto row_at = [&](uint32_t m, int r) -> uint64_t {
        const uint64_t gi = (uint64_t)m * kBM + r;
        return gi < p.rows ? rowpart(p.out_i0 + gi, p.out_geom) : kNoCol;
    };
    // container offset of output column n*W + jb + j; vec: j..j+3 is one aligned
    // 16-byte run of a tile row
    auto col_at = [&](uint32_t n, int j, bool& vec) -> uint64_t {
        const uint64_t gj = (uint64_t)n * W + jb + j;
        if (gj >= p.cols) {
            vec = false;
            return kNoCol;
        }
        uint64_t b, r;
        tdivmod(p.out_j0 + gj, p.out_geom, b, r);
        vec = p.vec_ok && (r & 3) == 0 && r + 3 < p.out_geom.t && gj + 3 < p.cols;
        return p.out_geom.shift >= 0 ? (dilate32(b) << (2 * p.out_geom.shift)) | r
                                     : dilate32(b) * p.out_geom.tt + r;
    };
    // edge path (a lane whose 4-column run is not one aligned 16-byte run): the
    // pass's rows element by element, staged through the transpose buffer
    // The lane's 4 column offsets of pass h are computed once (they do not depend on the
    // row), and a lane whose run lies wholly past the view (the right-edge tiles of a view
    // that is not a multiple of 128 wide) skips the rows at once.
    auto edge_cols = [&](uint32_t n, int h, uint64_t (&cc)[4]) -> bool {
        bool any = false;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            bool unused;
            cc[e] = col_at(n, PW * h + 4 * ch + e, unused);
            any |= cc[e] != kNoCol;
        }
        return any;
    };
    auto edge_load = [&](uint32_t m, uint32_t n, int h) {
        uint64_t cc[4];
        const bool any = edge_cols(n, h, cc);
#pragma unroll 1
        for (int i = 0; i < NI; ++i) {
            const uint64_t rb = any ? row_at(m, quad * 32 + RPI * i + sr) : kNoCol;
            const uint32_t dst = xaddr(RPI * i + sr, ch);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                sts32(dst + 4 * e, (rb != kNoCol && cc[e] != kNoCol) ? p.out[rb + cc[e]] : 0u);
        }
    };
    auto edge_store = [&](uint32_t m, uint32_t n, int h) {
        uint64_t cc[4];
        if (!edge_cols(n, h, cc)) return;
#pragma unroll 1
        for (int i = 0; i < NI; ++i) {
            const uint64_t rb = row_at(m, quad * 32 + RPI * i + sr);
            if (rb == kNoCol) continue;
            const uint32_t src = xaddr(RPI * i + sr, ch);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (cc[e] != kNoCol) p.out[rb + cc[e]] = lds32(src + 4 * e);
        }
    };
    for (uint32_t tile = first_tile; tile < num_tiles; tile += tile_stride) {
        const long long tp0 = diag_clock();
        uint32_t tm, n;
        tile_coords(tile, row_groups, p.Nt, p.group, tm, n);
        const uint32_t m = PAIR ? 2 * tm + rank : tm;
        uint32_t cur[WH];
        uint64_t rbase = 0;
        bool row_ok = false;
        const uint64_t* col = s_col + jb;
        // C_old of this tile (XPOSE): pass 0 by cp.async into the transpose buffer, pass 1
        // into registers; issued after the tile's last TMEM release and the final fold
        // (issuing them earlier -- at tile start, or between the two drain phases --
        // measured slower, profiles/r02_short_k.txt)
        uint4 c1[XPOSE ? NI : 1];
        uint32_t m1 = 0;
        uint64_t own = 0, c0[XPOSE ? NH : 1], rbs[XPOSE ? NI : 1];
        bool vec[XPOSE ? NH : 1];
        auto issue_cold0 = [&]() {
            if constexpr (XPOSE) {
                own = row_at(m, row);
#pragma unroll
                for (int h = 0; h < NH; ++h) c0[h] = col_at(n, PW * h + 4 * ch, vec[h]);
                // container offsets of the rows this lane moves in the coalesced order
#pragma unroll
                for (int i = 0; i < NI; ++i) rbs[i] = __shfl_sync(0xffffffffu, own, RPI * i + sr);
                if (p.mode != 2) {
#pragma unroll
                    for (int i = 0; i < NI; ++i) {
                        const uint64_t rb = rbs[i];
                        const bool live = rb != kNoCol;
                        if (vec[0])
                            cp_async16(xaddr(RPI * i + sr, ch), p.out + (live ? rb + c0[0] : 0), live ? 16u : 0u);
                    }
                    cp_async_commit();
                }
            }
        };
        auto issue_cold1 = [&]() {
            if constexpr (XPOSE) {
                if (p.mode != 2) {
#pragma unroll
                    for (int i = 0; i < NI; ++i) {
                        const bool ok = vec[1] && rbs[i] != kNoCol;
                        m1 |= (uint32_t)ok << i;
                        c1[i] = c_load(reinterpret_cast<const uint4*>(p.out + (ok ? rbs[i] + c0[1] : 0)));
                    }
                }
            }
        };
        bool cold0_issued = false, cold1_issued = false;
        auto issue_cold = [&]() {
            if (!cold0_issued) issue_cold0();
            if (!cold1_issued) issue_cold1();
        };
        if constexpr (XPOSE) {
            // the classes are folded from zero; C_old is loaded only after the tile's
            // (last) TMEM release, so its latency overlaps the next job's MMAs
#pragma unroll
            for (int j = 0; j < WH; ++j) cur[j] = 0u;
        } else {
            const uint64_t gi = (uint64_t)m * kBM + row;
            row_ok = gi < p.rows;
            rbase = row_ok ? __ldg(p.out_rowoff + gi) : 0;
            epi_bar_sync<EPI_THREADS>();  // previous tile's readers of s_col are done
            for (int j = ew * 32 + lane; j < W; j += EPI_THREADS) {
                const uint64_t gj = (uint64_t)n * W + j;
                s_col[j] = gj < p.cols ? __ldg(p.out_coloff + gj) : kNoCol;
            }
            epi_bar_sync<EPI_THREADS>();
            if (p.mode != 2 && row_ok) {
#pragma unroll
                for (int g = 0; g < WH / 4; ++g) {
                    const uint64_t c0 = col[4 * g], c3 = col[4 * g + 3];
                    if (p.vec_ok && c3 == c0 + 3 && (c0 & 3) == 0) {
                        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(p.out + rbase + c0));
                        cur[4 * g] = v.x;
                        cur[4 * g + 1] = v.y;
                        cur[4 * g + 2] = v.z;
                        cur[4 * g + 3] = v.w;
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint64_t cc = col[4 * g + e];
                            cur[4 * g + e] = cc != kNoCol ? p.out[rbase + cc] : 0u;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < WH; ++j) cur[j] = 0u;
            }
        }
        epi_pro += diag_clock() - tp0;
        for (uint32_t c = 0; c < nchunks; ++c) {
            const long long w0 = diag_clock();
            mbar_wait_hint(tmem_full, acc_ph, p.wait_hint);
            const long long w1 = diag_clock();
            epi_wait += w1 - w0;
            tc_fence_after();
            if constexpr (PAIR) {
#pragma unroll
                for (int j0 = 0; j0 < WH; j0 += CW) {
                    const bool live = (uint64_t)n * W + jb + j0 < p.cols;  // warp-uniform
                    int32_t acc[CLASSES][CW];
#pragma unroll
                    for (int k = 0; k < CLASSES; ++k)
                        tmem_ld<CW>(tmem + lane_base + k * W + jb + j0, acc[k]);
                    tmem_wait_ld();
#pragma unroll
                    for (int k = L; k < CLASSES; ++k) tmem_zero<CW>(tmem + lane_base + k * W + jb + j0);
                    if (live) {
#pragma unroll
                        for (int j = 0; j < CW; ++j) {
                            const uint32_t r = fold_classes<L, CW>(acc, j, p);
                            const uint32_t sum = cur[j0 + j] + r;
                            cur[j0 + j] = sum >= p.q ? sum - p.q : sum;
                        }
                    }
                }
                tmem_wait_st();
                release();
                epi_busy += diag_clock() - w1;
            } else {
                // Jobs alternate TMEM bases 0 / W.  The next job (other base) needs
                // this job's classes [1, C) (base 0) or [0, C-1) (base W) plus the
                // free region, so those are drained and folded first, TMEM is
                // released, and the remaining class is drained while the next
                // job's MMAs run.
                // lean folds (FOLD 1 / 2) exist only for w16 < 256: always the alternating layout
                const bool alt = (L == 2 && FOLD <= 2) || early_release<L>(p);
                const uint32_t tb = tmem + lane_base + ((alt && acc_ph) ? W : 0) + jb;
                if (!alt) {
                    // fixed layout: drain and fold every class, then release
                    drain(std::integral_constant<int, 0>{}, std::integral_constant<int, CLASSES>{}, tb, n, cur);
                    release();
                    epi_busy += diag_clock() - w1;
                    acc_ph ^= 1;
                    continue;
                }
                if constexpr (L == 2) {
                    // lean split for q = 2^16 - small (e.g. 65521): the first group
                    // leaves cur unreduced (< 2^32 - 2^24); the second group finishes
                    long long t_rel = 0;
                    drain_l2_small(tb, n, cur, acc_ph, [&]() {
                        t_rel = diag_clock();
#if MHG_COLD_MID
                        if constexpr (XPOSE) {
                            if (c + 1 == nchunks) {
                                issue_cold0();
                                cold0_issued = true;
                                if constexpr (MHG_COLD_MID >= 2) {
                                    issue_cold1();  // pass 1 too: its registers ride through the second drain
                                    cold1_issued = true;
                                }
                            }
                        }
#endif
                    });
                    // diagnostics: busy = the first drain group up to the TMEM release (what the
                    // next job's MMAs wait for); the second group + C_old issue go to epi_ldw
                    const long long t_end = diag_clock();
                    epi_busy += t_rel - w1;
                    epi_ldw += t_end - t_rel;
                    acc_ph ^= 1;
                    continue;
                }
                if (acc_ph == 0) {
                    drain(std::integral_constant<int, 1>{}, std::integral_constant<int, CLASSES>{}, tb, n, cur);
                    release();
                    epi_busy += diag_clock() - w1;
                    drain(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{}, tb, n, cur);
                } else {
                    drain(std::integral_constant<int, 0>{}, std::integral_constant<int, CLASSES - 1>{}, tb, n, cur);
                    release();
                    epi_busy += diag_clock() - w1;
                    drain(std::integral_constant<int, CLASSES - 1>{}, std::integral_constant<int, CLASSES>{}, tb, n, cur);
                }
            }
            acc_ph ^= 1;
        }
        const long long tt0 = diag_clock();
        if constexpr (XPOSE) {
            // out = (folded product + C_old) mod q.  The product is final here (< q <=
            // 2^16: XPOSE tiles are the <= 2-limb ones), so it is held two per register
            // while this tile's C_old loads are in flight -- they were issued only now,
            // after the last TMEM release, so their latency overlaps the next job's
            // MMAs.  Per pass: C_old staged into the buffer (coalesced order), read back
            // in row order and added, the sums written back in place, then stored in
            // the coalesced order.
            static_assert(NH == 2, "two column passes per epilogue warp");
            uint32_t c16[WH / 2];
#pragma unroll
            for (int j = 0; j < WH / 2; ++j) c16[j] = cur[2 * j] | (cur[2 * j + 1] << 16);
            const bool addc = p.mode != 2;
            issue_cold();
            const long long ta = diag_clock();
            epi_issue += ta - tt0;
            // The shared-memory loads of a pass are issued as one batch (the asm volatile
            // accesses keep source order, so load / use / store per chunk would expose every
            // load's latency: K = 1024 -1.3%).
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                if (addc) {
                    if (h == 0) {
                        if (!vec[0]) edge_load(m, n, 0);
                        cp_async_wait_all();
                        epi_land += diag_clock() - ta;
                    } else if (vec[1]) {
#pragma unroll
                        for (int i = 0; i < NI; ++i)
                            sts128(xaddr(RPI * i + sr, ch), ((m1 >> i) & 1u) ? c1[i] : make_uint4(0u, 0u, 0u, 0u));
                    } else {
                        edge_load(m, n, 1);
                    }
                    __syncwarp();
                }
                uint4 v[CPR];
#pragma unroll
                for (int g = 0; g < CPR; ++g) v[g] = addc ? lds128(xaddr(lane, g)) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int g = 0; g < CPR; ++g) {
                    const uint32_t w[4] = {v[g].x, v[g].y, v[g].z, v[g].w};
                    uint32_t o[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int jj = PW * h + 4 * g + e;
                        const uint32_t x = ((c16[jj >> 1] >> (16 * (jj & 1))) & 0xffffu) + w[e];
                        o[e] = umin(x, x - p.q);  // x < 2q
                    }
                    sts128(xaddr(lane, g), make_uint4(o[0], o[1], o[2], o[3]));
                }
                __syncwarp();
                static_assert(NI == CPR, "one transpose buffer row per lane");
#pragma unroll
                for (int i = 0; i < NI; ++i) v[i] = lds128(xaddr(RPI * i + sr, ch));
#pragma unroll
                for (int i = 0; i < NI; ++i)
                    if (vec[h] && rbs[i] != kNoCol) c_store(reinterpret_cast<uint4*>(p.out + rbs[i] + c0[h]), v[i]);
                if (!vec[h]) edge_store(m, n, h);
                __syncwarp();
            }
        } else if (row_ok) {
#pragma unroll
            for (int g = 0; g < WH / 4; ++g) {
                const uint64_t c0 = col[4 * g], c3 = col[4 * g + 3];
                if (p.vec_ok && c3 == c0 + 3 && (c0 & 3) == 0) {
                    __stcs(reinterpret_cast<uint4*>(p.out + rbase + c0),
                           make_uint4(cur[4 * g], cur[4 * g + 1], cur[4 * g + 2], cur[4 * g + 3]));
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint64_t cc = col[4 * g + e];
                        if (cc != kNoCol) p.out[rbase + cc] = cur[4 * g + e];
                    }
                }
            }
        }
        epi_tail += diag_clock() - tt0;
    }
    if (p.stats && warp == EW0 && lane == 0) {
        p.stats[(uint64_t)blockIdx.x * kStatCount + kStatEpiWaitFull] = epi_wait;
        p.stats[(uint64_t)blockIdx.x * kStatCount + kStatEpiBusy] = epi_busy;
        p.stats[(uint64_t)blockIdx.x * kStatCount + kStatEpiPrologue] = epi_pro;
        p.stats[(uint64_t)blockIdx.x * kStatCount + kStatEpiTail] = epi_tail;
        p.stats[(uint64_t)blockIdx.x * kStatCount + kStatEpiLdWait] = epi_ldw;
        p.stats[(uint64_t)blockIdx.x * kStatCount + kStatEpiIssue] = epi_issue;
        p.stats[(uint64_t)blockIdx.x * kStatCount + kStatEpiLand] = epi_land;
    }
}

template <int L, int FOLD = 3, bool NARROW = false>
__global__ void __launch_bounds__(GemmCfg<L, NARROW>::THREADS, 1) k_gemm(const GemmParams p) {
    using Cfg = GemmCfg<L, NARROW>;
    constexpr int W = Cfg::W;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
    uint64_t* s_col = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE + 256);  // W column offsets
    uint8_t* xbuf = reinterpret_cast<uint8_t*>(s_col + W);  // per-warp C transpose buffers

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t num_tiles = p.Mt * p.Nt;
    const uint32_t first_tile = blockIdx.x;
    const uint32_t tile_stride = gridDim.x;
    const uint32_t nchunks = (p.Kt + p.KC - 1) / p.KC;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, Cfg::EPI_WARPS);  // one arrive per epilogue warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // launched with programmatic stream serialisation: everything above overlapped the
    // previous kernel (the packs); operands and C may be read only after it completed
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp < Cfg::EPI_W0) {
#if MHG_SMR
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(MHG_SMR_CTL_REGS));
#endif
    if (warp == 0) {
        // ---------------- producer: one bulk copy per operand per stage
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            long long wait_empty = 0;
            uint32_t ord = 0;
            // lhs panels of the raster group are re-read by the next waves (evict_last),
            // rhs panels only by the current one (evict_first): -1.3% at n = 16384
            const uint64_t pol_keep = l2_policy_evict_last();
            const uint64_t pol_stream = p.keep_b ? pol_keep : l2_policy_evict_first();
            for (uint32_t tile = first_tile; tile < num_tiles; tile += tile_stride, ++ord) {
                uint32_t m, n;
                tile_coords(tile, p.Mt, p.Nt, p.group, m, n);
                const int8_t* a_src = p.apack + (uint64_t)m * p.Kt * Cfg::A_STAGE;
                const int8_t* b_src = p.bpack + (uint64_t)n * p.Kt * Cfg::B_STAGE;
                // serpentine K: odd tiles of a CTA sweep K backwards, so the next wave
                // starts on the panel slices the previous wave just left in L2
                const bool rev = ord & 1;
                for (uint32_t j = 0; j < p.Kt; ++j) {
                    const uint32_t kt = rev ? p.Kt - 1 - j : j;
                    const long long w0 = diag_clock();
                    mbar_wait_hint(&empty[st], ph ^ 1, p.wait_hint);
                    wait_empty += diag_clock() - w0;
                    mbar_expect_tx(&full[st], Cfg::STAGE);
                    bulk_g2s_hint(sA + st * Cfg::A_STAGE, a_src + (uint64_t)kt * Cfg::A_STAGE,
                                  Cfg::A_STAGE, &full[st], pol_keep);
                    bulk_g2s_hint(sB + st * Cfg::B_STAGE, b_src + (uint64_t)kt * Cfg::B_STAGE,
                                  Cfg::B_STAGE, &full[st], pol_stream);
                    if (++st == STAGES) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
            if (p.stats) p.stats[(uint64_t)blockIdx.x * kStatCount + kStatProdWaitEmpty] = wait_empty;
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread)
        if (lane == 0) {
            const uint32_t um = p.udig ? ~idesc_sign_mask() : ~0u;
            const uint32_t id_full = idesc_i8(kBM, Cfg::NB) & um;
            const uint32_t id_head = idesc_i8(kBM, (L > 1 ? L - 1 : 1) * W) & um;
            const uint32_t id_one = idesc_i8(kBM, W) & um;
            const bool alt_layout = early_release<L>(p);
            int st = 0;
            uint32_t ph = 0, acc_ph = 0;
            long long wait_full = 0, wait_tmem = 0;
            const long long t_begin = diag_clock();
            for (uint32_t tile = first_tile; tile < num_tiles; tile += tile_stride) {
                for (uint32_t c = 0; c < nchunks; ++c) {
                    const uint32_t kb = c * p.KC;
                    const uint32_t ke = (kb + p.KC < p.Kt) ? kb + p.KC : p.Kt;
                    long long w0 = diag_clock();
                    mbar_wait_hint(tmem_empty, acc_ph ^ 1, p.wait_hint);
                    wait_tmem += diag_clock() - w0;
                    tc_fence_after();
                    for (uint32_t kt = kb; kt < ke; ++kt) {
                        w0 = diag_clock();
                        mbar_wait_hint(&full[st], ph, p.wait_hint);
                        wait_full += diag_clock() - w0;
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + st * Cfg::A_STAGE);
                        const uint32_t b0 = smem_u32(sB + st * Cfg::B_STAGE);
#pragma unroll
                        for (int kk = 0; kk < kBK / 32; ++kk) {
                            const bool first = (kt == kb) && (kk == 0);
                            const uint64_t bd = sdesc(b0 + kk * 32);
#pragma unroll
                            for (int s = 0; s < L; ++s) {
                                const uint64_t ad = sdesc(a0 + s * kBM * kBK + kk * 32);
                                // accumulation jobs alternate TMEM bases 0 / W where the
                                // epilogue uses the early release (see epilogue_role)
                                const uint32_t d = tmem + ((alt_layout && acc_ph) ? W : 0) + s * W;
                                if (!first) {
                                    mma_i8(d, ad, bd, id_full, 1u);
                                } else if (s == 0) {
                                    mma_i8(d, ad, bd, id_full, 0u);
                                } else {
                                    // classes s..s+L-2 already hold a product; class
                                    // s+L-1 is touched for the first time
                                    mma_i8(d, ad, bd, id_head, 1u);
                                    mma_i8(d + (L - 1) * W, ad,
                                           sdesc(b0 + (L - 1) * W * kBK + kk * 32), id_one, 0u);
                                }
                            }
                        }
                        tc_commit(&empty[st]);
                        if (++st == STAGES) {
                            st = 0;
                            ph ^= 1;
                        }
                    }
                    tc_commit(tmem_full);
                    acc_ph ^= 1;
                }
            }
            if (p.stats) {
                unsigned long long* o = p.stats + (uint64_t)blockIdx.x * kStatCount;
                o[kStatTotal] = diag_clock() - t_begin;
                o[kStatMmaWaitFull] = wait_full;
                o[kStatMmaWaitTmem] = wait_tmem;
            }
        }
    }
    } else {
        // the inc must dominate the epilogue code for ptxas to allocate it the larger budget
#if MHG_SMR
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(MHG_SMR_EPI_REGS));
#endif
        epilogue_role<L, W, Cfg::EPI_WARPS, false, Cfg::XPOSE, FOLD, Cfg::EPI_W0>(
            p, first_tile, tile_stride, num_tiles, p.Mt, 0u, nchunks, tmem, s_col, tmem_full,
            tmem_empty, warp, lane, xbuf);
    }

    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// =====================================================================
// K3' k_gemm2: the same GEMM on a CTA pair (tcgen05 cta_group::2, M = 256).
// Each CTA of the pair holds its own 128-row A tile (all L limbs) and HALF of
// the stacked B' (N rows [rank*NB/2, (rank+1)*NB/2)); the leader issues one
// 256 x NB x 32 MMA per limb that reads both CTAs' shared memory and writes
// each CTA's TMEM (its 128 rows).  Per-SM operand traffic drops by 25%
// versus k_gemm (B' is no longer replicated per 128 rows).
//   - loads: cp.async.bulk.tensor.2d.cta_group::2 from both CTAs complete on
//     the LEADER's full barrier (mapa address);
//   - MMA completion: tcgen05.commit.cta_group::2 multicast to both CTAs'
//     empty / tmem_full barriers;
//   - TMEM release: each epilogue warp of both CTAs arrives on the leader's
//     tmem_empty (remote arrive through the cluster window);
//   - the upper weight classes [L, 2L-1) are zeroed by the epilogue right
//     after it drains them, so every MMA but the first of a chunk accumulates.
// =====================================================================
template <int L>
struct Gemm2Cfg {
    static constexpr int W = (L <= 2) ? 128 : 64;
    static constexpr int NB = L * W;      // UMMA N of one limb MMA (stacked B')
    static constexpr int NBR = L * W;     // B' rows per (column tile, k tile)
    static constexpr int NBH = NBR / 2;   // B' rows per CTA
    static constexpr int CLASSES = 2 * L - 1;
    static constexpr int A_STAGE = L * kBM * kBK;
    static constexpr int B_STAGE = NBH * kBK;
    static constexpr int STAGE = A_STAGE + B_STAGE;
    // row-per-thread C access (the coalesced transpose-buffer epilogue measured within
    // 1% for the 3- and 4-limb pairs, profiles/r01_pair_wide_primes.txt)
    static constexpr int STAGES_RAW = (220 * 1024) / STAGE;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static constexpr int SMEM = 1024 + STAGES * STAGE + 512 + 8 * W;
    static_assert(SMEM <= 232448, "227 KB dynamic shared memory limit");
    static constexpr int EPI_WARPS = 8;
    static constexpr int EPI_THREADS = EPI_WARPS * 32;
    static constexpr int WH = W / 2;
    static constexpr int THREADS = 64 + EPI_THREADS;
    static_assert(CLASSES * W <= 512, "TMEM columns");
    static_assert(STAGES >= 2, "pipeline depth");
    static_assert(NBH % 16 == 0 || NBH == 64, "B' half rows");
};

template <int L>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Gemm2Cfg<L>::THREADS, 1)
    k_gemm2(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap tmA,
            const __grid_constant__ CUtensorMap tmB) {
    using Cfg = Gemm2Cfg<L>;
    constexpr int W = Cfg::W;
    constexpr int WH = Cfg::WH;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
    uint64_t* s_col = tmem_empty + 2;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const uint32_t Mt2 = p.Mt >> 1;  // host pads Mt to even
    const uint32_t num_tiles = Mt2 * p.Nt;
    const uint32_t nchunks = (p.Kt + p.KC - 1) / p.KC;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 2 * Cfg::EPI_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // launched with programmatic stream serialisation: everything above overlapped the
    // previous kernel (the packs); operands and C may be read only after it completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (warp >= 2) {
        // zero the upper weight classes once; afterwards the epilogue re-zeroes
        // them as it drains them
        const int ew = warp - 2, quad = warp & 3, jb = (ew >> 2) * WH;
        const uint32_t lb = (uint32_t)(quad * 32) << 16;
#pragma unroll
        for (int k = L; k < Cfg::CLASSES; ++k)
#pragma unroll
            for (int j0 = 0; j0 < WH; j0 += 16) tmem_zero16(tmem + lb + k * W + jb + j0);
        tmem_wait_st();
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();

    if (warp == 0) {
        if (lane == 0) {
            long long wait_empty = 0;
            int st = 0;
            uint32_t ph = 0;
            uint32_t ord = 0;
            for (uint32_t tile = pair; tile < num_tiles; tile += npairs, ++ord) {
                uint32_t pm, n;
                tile_coords(tile, Mt2, p.Nt, p.group, pm, n);
                const uint32_t m = 2 * pm + rank;
                const bool rev = ord & 1;
                for (uint32_t j = 0; j < p.Kt; ++j) {
                    const uint32_t kt = rev ? p.Kt - 1 - j : j;
                    const long long w0 = diag_clock();
                    mbar_wait(&empty[st], ph ^ 1);
                    wait_empty += diag_clock() - w0;
                    if (rank == 0) mbar_expect_tx(&full[st], 2 * Cfg::STAGE);
                    const uint32_t lbar = mapa_shared(smem_u32(&full[st]), 0);
                    const int arow = (int)(((uint64_t)m * p.Kt + kt) * L * kBM);
#pragma unroll
                    for (int l = 0; l < L; ++l)
                        tma2d_pair(smem_u32(sA + st * Cfg::A_STAGE + l * kBM * kBK), &tmA, 0,
                                   arow + l * kBM, lbar);
                    const int brow = (int)(((uint64_t)n * p.Kt + kt) * Cfg::NBR + rank * Cfg::NBH);
                    tma2d_pair(smem_u32(sB + st * Cfg::B_STAGE), &tmB, 0, brow, lbar);
                    if (++st == STAGES) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
            if (p.stats) p.stats[(uint64_t)blockIdx.x * kStatCount + kStatProdWaitEmpty] = wait_empty;
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            const uint32_t id_full = idesc_i8(2 * kBM, Cfg::NB) & (p.udig ? ~idesc_sign_mask() : ~0u);
            int st = 0;
            uint32_t ph = 0, job = 0;
            long long wait_full = 0, wait_tmem = 0;
            const long long t_begin = diag_clock();
            for (uint32_t tile = pair; tile < num_tiles; tile += npairs) {
                for (uint32_t c = 0; c < nchunks; ++c, ++job) {
                    const uint32_t kb = c * p.KC;
                    const uint32_t ke = (kb + p.KC < p.Kt) ? kb + p.KC : p.Kt;
                    long long w0 = diag_clock();
                    mbar_wait(tmem_empty, (job & 1) ^ 1);
                    wait_tmem += diag_clock() - w0;
                    tc_fence_after();
                    const uint32_t dbase = tmem;
                    for (uint32_t kt = kb; kt < ke; ++kt) {
                        w0 = diag_clock();
                        mbar_wait(&full[st], ph);
                        wait_full += diag_clock() - w0;
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + st * Cfg::A_STAGE);
                        const uint32_t b0 = smem_u32(sB + st * Cfg::B_STAGE);
#pragma unroll
                        for (int kk = 0; kk < kBK / 32; ++kk) {
                            const bool first = (kt == kb) && (kk == 0);
#pragma unroll
                            for (int s = 0; s < L; ++s) {
                                mma_i8_pair(dbase + s * W, sdesc(a0 + s * kBM * kBK + kk * 32),
                                            sdesc(b0 + kk * 32), id_full, (first && s == 0) ? 0u : 1u);
                            }
                        }
                        tc_commit_pair(&empty[st]);
                        if (++st == STAGES) {
                            st = 0;
                            ph ^= 1;
                        }
                    }
                    tc_commit_pair(tmem_full);
                }
            }
            if (p.stats) {
                unsigned long long* o = p.stats + (uint64_t)blockIdx.x * kStatCount;
                o[kStatTotal] = diag_clock() - t_begin;
                o[kStatMmaWaitFull] = wait_full;
                o[kStatMmaWaitTmem] = wait_tmem;
            }
        }
    } else {
        epilogue_role<L, W, Cfg::EPI_WARPS, true, false, 3>(
            p, pair, npairs, num_tiles, Mt2, rank, nchunks, tmem, s_col, tmem_full, tmem_empty, warp,
            lane);
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// Kernel launch with programmatic stream serialisation (PDL): the kernel may begin before
// the previous kernel in the stream completes and waits for it with griddepcontrol.wait.
// Used for GEMMs of at most one wave of tiles (cfg1-class problems: the launch and prologue
// are a large part of the kernel, -10% per step); multi-wave GEMMs launch plainly (the TU
// sweep measured 2.7% slower with PDL on every step, profiles/r02b/README.md).
template <typename... KArgs, typename... Args>
int launch_pdl(bool pdl, void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
               Args&&... args) {
    if (!pdl) {
        kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
        return (int)cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int L>
int launch_gemm2_t(const GemmParams& p, const void* tmA, const void* tmB, int num_sms,
                   cudaStream_t s) {
    using Cfg = Gemm2Cfg<L>;
    const uint32_t tiles = (p.Mt / 2) * p.Nt;
    uint32_t grid = 2 * tiles < (uint32_t)num_sms ? 2 * tiles : (uint32_t)num_sms;
    grid &= ~1u;
    return launch_pdl(tiles * 2 <= (uint32_t)num_sms, k_gemm2<L>, grid, Cfg::THREADS, Cfg::SMEM, s, p, *static_cast<const CUtensorMap*>(tmA),
                      *static_cast<const CUtensorMap*>(tmB));
}

template <int L>
int configure_gemm2_t() {
    return (int)cudaFuncSetAttribute(k_gemm2<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Gemm2Cfg<L>::SMEM);
}

template <int L>
int configure_gemm_t() {
    int e = (int)cudaFuncSetAttribute(k_gemm<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      GemmCfg<L>::SMEM);
    if constexpr (L <= 2) {
        using N = GemmCfg<L, true>;
        if (!e) e = (int)cudaFuncSetAttribute(k_gemm<L, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, N::SMEM);
    }
    if constexpr (L == 2) {
        using N = GemmCfg<L, true>;
        if (!e)
            e = (int)cudaFuncSetAttribute(k_gemm<L, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          GemmCfg<L>::SMEM);
        if (!e)
            e = (int)cudaFuncSetAttribute(k_gemm<L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          GemmCfg<L>::SMEM);
        if (!e) e = (int)cudaFuncSetAttribute(k_gemm<L, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, N::SMEM);
        if (!e) e = (int)cudaFuncSetAttribute(k_gemm<L, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, N::SMEM);
    }
    return e;
}

// Writes `value` into every cell of a view (SET with an empty inner dimension).
__global__ void k_fill_view(uint32_t* __restrict__ out, const uint64_t* __restrict__ rowoff,
                            const uint64_t* __restrict__ coloff, uint64_t rows, uint64_t cols,
                            uint32_t value) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < rows * cols;
         x += (uint64_t)gridDim.x * blockDim.x)
        out[rowoff[x / cols] + coloff[x % cols]] = value;
}

template <int L, bool NARROW>
int launch_gemm_cfg(const GemmParams& p, int num_sms, cudaStream_t s) {
    using Cfg = GemmCfg<L, NARROW>;
    const uint32_t tiles = p.Mt * p.Nt;
    const int grid = (int)(tiles < (uint32_t)num_sms ? tiles : (uint32_t)num_sms);
    const bool one_wave = tiles <= (uint32_t)num_sms;
    if constexpr (L == 2) {
        if (p.fold == 1 || p.fold == 2) {
            if (p.fold == 1) return launch_pdl(one_wave, k_gemm<L, 1, NARROW>, grid, Cfg::THREADS, Cfg::SMEM, s, p);
            return launch_pdl(one_wave, k_gemm<L, 2, NARROW>, grid, Cfg::THREADS, Cfg::SMEM, s, p);
        }
    }
    return launch_pdl(one_wave, k_gemm<L, 3, NARROW>, grid, Cfg::THREADS, Cfg::SMEM, s, p);
}

template <int L>
int launch_gemm_t(const GemmParams& p, int num_sms, cudaStream_t s) {
    if constexpr (L <= 2) {
        if (p.narrow) return launch_gemm_cfg<L, true>(p, num_sms, s);
    }
    return launch_gemm_cfg<L, false>(p, num_sms, s);
}

template <int L>
int launch_pack_t(int trans, const uint32_t* src, const uint64_t* rowoff, const uint64_t* coloff,
                  int vecok, uint64_t R, uint64_t K, uint32_t rpt, uint32_t Rtiles, uint32_t Kt,
                  int8_t* dst, DigitParams dp, cudaStream_t s) {
    const uint64_t Rpad = (uint64_t)Rtiles * rpt;
    if (trans) {
        const uint64_t blocks = ((Rpad + 127) / 128) * Kt * (kBK / 32);
        k_pack_cols<L><<<(unsigned)blocks, 256, 0, s>>>(src, rowoff, coloff, vecok, R, K, rpt, Kt,
                                                        Rpad, dst, dp);
    } else {
        const uint64_t blocks = (Rpad / 32) * (((uint64_t)Kt * kBK + kPackK - 1) / kPackK);
        k_pack_rows<L><<<(unsigned)blocks, 256, 0, s>>>(src, rowoff, coloff, vecok, R, K, rpt, Kt,
                                                        Rpad, dst, dp);
    }
    return (int)cudaGetLastError();
}

}  // namespace

int launch_offsets(uint64_t* dst, uint64_t start, uint64_t count, TileGeom g, int is_row,
                   void* stream) {
    if (count == 0) return 0;
    const unsigned blocks = (unsigned)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
    k_offsets<<<blocks, 256, 0, (cudaStream_t)stream>>>(dst, start, count, g, is_row);
    return (int)cudaGetLastError();
}

// LDG/STG conversion kernels: Morton-order iteration (k_conv_z, 4 groups in flight per
// thread, 0.84-0.89 of measured HBM, profiles/r01_conversion.txt) where the row-major
// buffer is 16-byte aligned and t is a power of two with t % 4 == 0 (morton = 1), else
// the element-wise row-order kernels.
int launch_rm_to_mh(const uint32_t* rm, uint32_t* mh, uint64_t n, TileGeom g, uint32_t q,
                    int* bad_flag, int morton, void* stream) {
    const bool aligned = (reinterpret_cast<uintptr_t>(rm) & 15) == 0;
    const bool z = morton && aligned && g.shift >= 0 && g.t % 4 == 0;
    if (z) k_conv_z<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(rm, mh, n, g, q, bad_flag, 1);
    else k_rm_to_mh<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(rm, mh, n, g, q, bad_flag);
    return (int)cudaGetLastError();
}

int launch_mh_to_rm(const uint32_t* mh, uint32_t* rm, uint64_t n, TileGeom g, int morton, void* stream) {
    const bool z = morton && ((reinterpret_cast<uintptr_t>(rm) & 15) == 0) && g.shift >= 0 && g.t % 4 == 0;
    if (z) k_conv_z<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(mh, rm, n, g, 0u, nullptr, 0);
    else k_mh_to_rm<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(mh, rm, n, g);
    return (int)cudaGetLastError();
}

template <int L>
int launch_pack_pair_t(PackArgs a, PackArgs b, cudaStream_t s) {
    a.Rpad = (uint64_t)a.Rtiles * a.rpt;
    b.Rpad = (uint64_t)b.Rtiles * b.rpt;
    const uint64_t na = (a.Rpad / 32) * (((uint64_t)a.Kt * kBK + kPackK - 1) / kPackK);
    const uint64_t nb = ((b.Rpad + 127) / 128) * b.Kt * (kBK / 32);
    k_pack_pair<L><<<(unsigned)(na + nb), 256, 0, s>>>(a, b, (uint32_t)na);
    return (int)cudaGetLastError();
}

int launch_pack_pair(int L, const PackArgs& lhs, const PackArgs& rhs, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (L) {
        case 1: return launch_pack_pair_t<1>(lhs, rhs, s);
        case 2: return launch_pack_pair_t<2>(lhs, rhs, s);
        case 3: return launch_pack_pair_t<3>(lhs, rhs, s);
        case 4: return launch_pack_pair_t<4>(lhs, rhs, s);
    }
    return (int)cudaErrorInvalidValue;
}

int launch_pack(int L, int trans, const uint32_t* src, const uint64_t* rowoff,
                const uint64_t* coloff, int vecok, uint64_t R, uint64_t K, uint32_t rpt,
                uint32_t Rtiles, uint32_t Kt, int8_t* dst, DigitParams dp, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (L) {
        case 1: return launch_pack_t<1>(trans, src, rowoff, coloff, vecok, R, K, rpt, Rtiles, Kt, dst, dp, s);
        case 2: return launch_pack_t<2>(trans, src, rowoff, coloff, vecok, R, K, rpt, Rtiles, Kt, dst, dp, s);
        case 3: return launch_pack_t<3>(trans, src, rowoff, coloff, vecok, R, K, rpt, Rtiles, Kt, dst, dp, s);
        case 4: return launch_pack_t<4>(trans, src, rowoff, coloff, vecok, R, K, rpt, Rtiles, Kt, dst, dp, s);
    }
    return (int)cudaErrorInvalidValue;
}

int launch_gemm(int L, const GemmParams& p, int num_sms, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (L) {
        case 1: return launch_gemm_t<1>(p, num_sms, s);
        case 2: return launch_gemm_t<2>(p, num_sms, s);
        case 3: return launch_gemm_t<3>(p, num_sms, s);
        case 4: return launch_gemm_t<4>(p, num_sms, s);
    }
    return (int)cudaErrorInvalidValue;
}

int configure_kernels() {
    {
        const int e = (int)cudaFuncSetAttribute(k_conv_tma<kConvUnits>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, conv_tma_smem());
        if (e) return e;
    }
    int e = configure_gemm_t<1>();
    if (!e) e = configure_gemm_t<2>();
    if (!e) e = configure_gemm_t<3>();
    if (!e) e = configure_gemm_t<4>();
    if (!e) e = configure_gemm2_t<1>();
    if (!e) e = configure_gemm2_t<2>();
    if (!e) e = configure_gemm2_t<3>();
    if (!e) e = configure_gemm2_t<4>();
    return e;
}

int launch_gemm2(int L, const GemmParams& p, const void* tmA, const void* tmB, int num_sms,
                 void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (L) {
        case 1: return launch_gemm2_t<1>(p, tmA, tmB, num_sms, s);
        case 2: return launch_gemm2_t<2>(p, tmA, tmB, num_sms, s);
        case 3: return launch_gemm2_t<3>(p, tmA, tmB, num_sms, s);
        case 4: return launch_gemm2_t<4>(p, tmA, tmB, num_sms, s);
    }
    return (int)cudaErrorInvalidValue;
}

int gemm2_b_box_rows(int L) { return (L <= 2 ? 128 : 64) * L / 2; }

int launch_fill_view(uint32_t* out, const uint64_t* rowoff, const uint64_t* coloff, uint64_t rows,
                     uint64_t cols, uint32_t value, void* stream) {
    if (rows == 0 || cols == 0) return 0;
    const uint64_t total = rows * cols;
    const unsigned blocks = (unsigned)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    k_fill_view<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, rowoff, coloff, rows, cols, value);
    return (int)cudaGetLastError();
}

// ------------------------------------------------------------ verification
// Freivalds' check of a finished multiply (mhg_verify): C_new r == C_old r +/- A (B r)
// (mod q) for random vectors r.  Every step is a row-wise mat-vec over a view, HBM-bound:
// one warp per view row, lanes striding the columns (coalesced inside Morton tile rows),
// 64-bit accumulation with a Barrett reduction per term.
__device__ __forceinline__ uint64_t mod64(uint64_t u, uint32_t q, uint64_t mu) {
    uint64_t r = u - __umul64hi(u, mu) * q;
    return r >= q ? r - q : r;
}

// y[i] = sum_j M[rowoff[i] + coloff[j]] x[j] mod q for i < rows
__global__ void k_matvec(const uint32_t* __restrict__ m, const uint64_t* __restrict__ rowoff,
                         const uint64_t* __restrict__ coloff, uint64_t rows, uint64_t cols,
                         const uint32_t* __restrict__ x, uint32_t* __restrict__ y, uint32_t q, uint64_t mu) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < rows; i += warps) {
        const uint32_t* row = m + rowoff[i];
        uint64_t acc = 0;
        for (uint64_t j = lane; j < cols; j += 32)
            acc = mod64(acc + (uint64_t)__ldcs(row + coloff[j]) * x[j], q, mu);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) y[i] = (uint32_t)mod64(acc, q, mu);
    }
}

// r[j] uniform-ish in [0, q) from (seed, j) (splitmix64)
__global__ void k_random_vec(uint32_t* __restrict__ r, uint64_t n, uint64_t seed, uint32_t q) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        r[j] = (uint32_t)(((unsigned __int128)z * q) >> 64);
    }
}

// mode 0: new == old + z, 1: new == old - z, 2: new == z; any mismatch sets *bad
__global__ void k_freivalds_cmp(const uint32_t* __restrict__ wn, const uint32_t* __restrict__ wo,
                                const uint32_t* __restrict__ z, uint64_t rows, uint32_t q, int mode,
                                int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t want;
        if (mode == 2) want = z[i];
        else if (mode == 0) want = (uint32_t)(((uint64_t)wo[i] + z[i]) % q);
        else want = (uint32_t)(((uint64_t)wo[i] + q - z[i]) % q);
        if (want != wn[i]) atomicOr(bad, 1);
    }
}

int launch_matvec(const uint32_t* m, const uint64_t* rowoff, const uint64_t* coloff, uint64_t rows,
                  uint64_t cols, const uint32_t* x, uint32_t* y, uint32_t q, int num_sms, void* stream) {
    if (rows == 0) return 0;
    const uint64_t mu = ~uint64_t(0) / q;
    const uint64_t blocks = (rows + 7) / 8;  // 8 warps per block
    const uint64_t cap = (uint64_t)(num_sms > 0 ? num_sms : 148) * 8;
    k_matvec<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, (cudaStream_t)stream>>>(m, rowoff, coloff, rows,
                                                                                        cols, x, y, q, mu);
    return (int)cudaGetLastError();
}

int launch_random_vec(uint32_t* r, uint64_t n, uint64_t seed, uint32_t q, void* stream) {
    if (n == 0) return 0;
    const uint64_t blocks = (n + 255) / 256;
    k_random_vec<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, (cudaStream_t)stream>>>(r, n, seed, q);
    return (int)cudaGetLastError();
}

int launch_freivalds_cmp(const uint32_t* wn, const uint32_t* wo, const uint32_t* z, uint64_t rows, uint32_t q,
                         int mode, int* bad, void* stream) {
    if (rows == 0) return 0;
    const uint64_t blocks = (rows + 255) / 256;
    k_freivalds_cmp<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, (cudaStream_t)stream>>>(wn, wo, z, rows, q,
                                                                                                 mode, bad);
    return (int)cudaGetLastError();
}

// 16-bit upload wire (mhg_matrix_upload, q <= 2^16): residues arrive as uint16 and
// are widened into the container.  HBM-bound: 6 B per cell (2 read + 4 written);
// 16-byte loads of 8 cells, two 16-byte stores, grid-stride.  A range upload may
// start anywhere: `head` cells are widened one by one until both pointers are
// 16-byte aligned (vec = 0: the whole range element-wise).
__global__ void k_widen16(const uint16_t* __restrict__ src, uint32_t* __restrict__ dst,
                          uint64_t count, uint32_t head, int vec) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (!vec) {
        for (uint64_t i = tid; i < count; i += stride) dst[i] = src[i];
        return;
    }
    if (tid < head) dst[tid] = src[tid];
    const uint64_t groups = (count - head) / 8;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    for (uint64_t g = tid; g < groups; g += stride) {
        const uint4 v = __ldcs(s4 + g);
        uint4 lo, hi;
        lo.x = v.x & 0xffffu; lo.y = v.x >> 16; lo.z = v.y & 0xffffu; lo.w = v.y >> 16;
        hi.x = v.z & 0xffffu; hi.y = v.z >> 16; hi.z = v.w & 0xffffu; hi.w = v.w >> 16;
        d4[2 * g] = lo;
        d4[2 * g + 1] = hi;
    }
    const uint64_t tail = head + groups * 8 + tid;
    if (tail < count) dst[tail] = src[tail];
}

int conv_tma_smem() { return kConvUnits * kConvUnitBytes + 1024; }

int launch_conv_tma(const void* tmap, uint32_t* mh, uint64_t n, TileGeom g, uint32_t q, int* bad,
                    int to_mh, int num_sms, void* stream) {
    uint32_t R = (uint32_t)g.t;
    while ((uint64_t)R * g.t * 4 > (uint64_t)kConvUnitBytes) R >>= 1;
    const int grid = kConvCtasPerSm * (num_sms > 0 ? num_sms : 148);
    const CUtensorMap& tm = *static_cast<const CUtensorMap*>(tmap);
    k_conv_tma<kConvUnits><<<grid, 128, conv_tma_smem(), (cudaStream_t)stream>>>(tm, mh, n, g, R, q, bad,
                                                                                 to_mh);
    return (int)cudaGetLastError();
}

int launch_widen16(const uint16_t* src, uint32_t* dst, uint64_t count, int num_sms, void* stream) {
    if (count == 0) return 0;
    const uint64_t mis = (reinterpret_cast<uintptr_t>(src) >> 1) & 7;
    uint32_t head = (uint32_t)((8 - mis) & 7);
    if (head > count) head = (uint32_t)count;
    const int vec = ((reinterpret_cast<uintptr_t>(src) & 1) == 0) &&
                    ((reinterpret_cast<uintptr_t>(dst + head) & 15) == 0);
    const uint64_t groups = (count + 7) / 8;
    uint64_t blocks = (groups + 255) / 256;
    const uint64_t cap = (uint64_t)(num_sms > 0 ? num_sms : 148) * 8;
    if (blocks > cap) blocks = cap;
    k_widen16<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(src, dst, count, head, vec);
    return (int)cudaGetLastError();
}

int diag_build() { return MHG_DIAG; }

int gemm_smem_bytes(int L) {
    switch (L) {
        case 1: return GemmCfg<1>::SMEM;
        case 2: return GemmCfg<2>::SMEM;
        case 3: return GemmCfg<3>::SMEM;
        case 4: return GemmCfg<4>::SMEM;
    }
    return 0;
}

}  // namespace mhg

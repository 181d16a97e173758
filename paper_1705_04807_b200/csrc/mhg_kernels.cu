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
#include <cuda_runtime.h>

#include <cstdint>

#include "mhg_internal.hpp"

namespace mhg {
namespace {

// ------------------------------------------------------------ index helpers
__device__ __forceinline__ uint64_t dilate32(uint64_t x) {
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
    return (dilate32(b) << 1) * g.tt + r * g.t;
}

__device__ __forceinline__ uint64_t colpart(uint64_t j, const TileGeom& g) {
    uint64_t b, r;
    tdivmod(j, g, b, r);
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
    const bool vec = (g.t % 4 == 0) && (n % 4 == 0);
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

__global__ void k_mh_to_rm(const uint32_t* __restrict__ mh, uint32_t* __restrict__ rm, uint64_t n,
                           TileGeom g) {
    const uint64_t groups = n * n / 4;
    const bool vec = (g.t % 4 == 0) && (n % 4 == 0);
    if (vec) {
        for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < groups;
             x += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t i = (4 * x) / n, j = (4 * x) % n;
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(mh + rowpart(i, g) + colpart(j, g)));
            __stcs(reinterpret_cast<uint4*>(rm) + x, v);
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
    int32_t x = v > dp.H ? (int32_t)(v - dp.q) : (int32_t)v;
#pragma unroll
    for (int s = 0; s < L - 1; ++s) {
        const int8_t lo = (int8_t)(x & 0xff);
        d[s] = lo;
        x = (x - (int32_t)lo) >> 8;
    }
    d[L - 1] = (int8_t)x;
}

constexpr int kPackStride = kBK + 4;  // smem row stride (bytes): conflict-free byte scatter

// One block = 32 pack rows x 128 K of one operand.  Output layout per
// (row tile, k tile): [L][rows_per_tile][128 B] with the SWIZZLE_128B
// pattern applied (16-byte chunk c of row r stored at chunk c ^ (r & 7)).
template <int L, bool TRANS>
__global__ void __launch_bounds__(256) k_pack(const uint32_t* __restrict__ src,
                                              const uint64_t* __restrict__ rowoff,
                                              const uint64_t* __restrict__ coloff, uint64_t R,
                                              uint64_t K, uint32_t rows_per_tile, uint32_t Kt,
                                              int8_t* __restrict__ dst, DigitParams dp) {
    __shared__ __align__(16) int8_t sd[L][kPackRows][kPackStride];
    const uint32_t kt = blockIdx.x % Kt;
    const uint64_t rb = blockIdx.x / Kt;
    const uint64_t pr0 = rb * kPackRows;
    const uint64_t k0 = (uint64_t)kt * kBK;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;

    if (!TRANS) {
        // lanes walk K (contiguous inside a Morton tile row of the source)
        uint64_t co[4];
        bool kok[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint64_t kk = k0 + tx + 32 * b;
            kok[b] = kk < K;
            co[b] = kok[b] ? __ldg(coloff + kk) : 0;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int r = ty + 8 * a;
            const uint64_t pr = pr0 + r;
            const bool rok = pr < R;
            const uint64_t ro = rok ? __ldg(rowoff + pr) : 0;
            uint32_t v[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) v[b] = (rok && kok[b]) ? __ldg(src + ro + co[b]) : 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                int8_t d[L];
                to_digits<L>(v[b], dp, d);
#pragma unroll
                for (int s = 0; s < L; ++s) sd[s][r][tx + 32 * b] = d[s];
            }
        }
    } else {
        // lanes walk pack rows = source columns (contiguous in the source)
        const uint64_t pr = pr0 + tx;
        const bool rok = pr < R;
        const uint64_t co = rok ? __ldg(coloff + pr) : 0;
#pragma unroll 4
        for (int b = 0; b < kBK / 8; ++b) {
            const int kloc = ty + 8 * b;
            const uint64_t kk = k0 + kloc;
            const bool kok = kk < K;
            const uint64_t ro = kok ? __ldg(rowoff + kk) : 0;
            const uint32_t v = (rok && kok) ? __ldg(src + ro + co) : 0u;
            int8_t d[L];
            to_digits<L>(v, dp, d);
#pragma unroll
            for (int s = 0; s < L; ++s) sd[s][tx][kloc] = d[s];
        }
    }
    __syncthreads();

    const uint64_t rtile = pr0 / rows_per_tile;
    const uint32_t rit0 = (uint32_t)(pr0 % rows_per_tile);
    int8_t* base = dst + ((rtile * Kt + kt) * (uint64_t)L) * rows_per_tile * kBK;
#pragma unroll
    for (int e = 0; e < L; ++e) {
        const int cid = threadIdx.x + 256 * e;  // L * 32 rows * 8 chunks
        const int s = cid >> 8, r = (cid >> 3) & 31, ch = cid & 7;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&sd[s][r][ch * 16]);
        const uint4 val = make_uint4(w[0], w[1], w[2], w[3]);
        const uint32_t rit = rit0 + r;
        int8_t* o = base + (uint64_t)s * rows_per_tile * kBK + (uint64_t)rit * kBK +
                    ((ch ^ (rit & 7)) << 4);
        *reinterpret_cast<uint4*>(o) = val;
    }
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

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
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

// K-major operand, SWIZZLE_128B: 8-row x 128-byte atoms, 1024 B apart (SBO).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;    // SBO
    d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;              // SWIZZLE_128B
    return d;
}

// kind::i8 instruction descriptor: s8 x s8 -> s32, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4)                   // D format S32
           | (1u << 7)                 // A signed
           | (1u << 10)                // B signed
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
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

template <int L>
struct GemmCfg {
    static constexpr int W = (L <= 2) ? 128 : 64;       // output columns per tile
    static constexpr int NB = L * W;                    // UMMA N of the stacked B'
    static constexpr int CLASSES = 2 * L - 1;           // weight classes 256^c
    static constexpr int A_STAGE = L * kBM * kBK;       // bytes
    static constexpr int B_STAGE = NB * kBK;            // bytes
    static constexpr int STAGE = A_STAGE + B_STAGE;
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE;
    static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
    static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE + 256 /*barriers*/;
    static constexpr int THREADS = 192;                 // producer, MMA, 4 epilogue warps
    static_assert(CLASSES * W <= 512, "TMEM columns");
    static_assert(STAGES >= 2, "pipeline depth");
};

__device__ __forceinline__ void tile_coords(uint32_t tile, uint32_t Mt, uint32_t Nt, uint32_t& m,
                                            uint32_t& n) {
    constexpr uint32_t G = 16;  // grouped raster: 16 row tiles share B panels in L2
    const uint32_t group = G * Nt;
    const uint32_t gid = tile / group;
    const uint32_t first_m = gid * G;
    const uint32_t gm = (Mt - first_m) < G ? (Mt - first_m) : G;
    const uint32_t local = tile - gid * group;
    m = first_m + local % gm;
    n = local / gm;
}

template <int L>
__global__ void __launch_bounds__(GemmCfg<L>::THREADS, 1) k_gemm(const GemmParams p) {
    using Cfg = GemmCfg<L>;
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

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t num_tiles = p.Mt * p.Nt;
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
        mbar_init(tmem_empty, 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer: one bulk copy per operand per stage
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                uint32_t m, n;
                tile_coords(tile, p.Mt, p.Nt, m, n);
                const int8_t* a_src = p.apack + (uint64_t)m * p.Kt * Cfg::A_STAGE;
                const int8_t* b_src = p.bpack + (uint64_t)n * p.Kt * Cfg::B_STAGE;
                for (uint32_t kt = 0; kt < p.Kt; ++kt) {
                    mbar_wait(&empty[st], ph ^ 1);
                    mbar_expect_tx(&full[st], Cfg::STAGE);
                    bulk_g2s(sA + st * Cfg::A_STAGE, a_src + (uint64_t)kt * Cfg::A_STAGE,
                             Cfg::A_STAGE, &full[st]);
                    bulk_g2s(sB + st * Cfg::B_STAGE, b_src + (uint64_t)kt * Cfg::B_STAGE,
                             Cfg::B_STAGE, &full[st]);
                    if (++st == STAGES) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread)
        if (lane == 0) {
            constexpr uint32_t id_full = idesc_i8(kBM, Cfg::NB);
            constexpr uint32_t id_head = idesc_i8(kBM, (L > 1 ? L - 1 : 1) * W);
            constexpr uint32_t id_one = idesc_i8(kBM, W);
            int st = 0;
            uint32_t ph = 0, acc_ph = 0;
            for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                for (uint32_t c = 0; c < nchunks; ++c) {
                    const uint32_t kb = c * p.KC;
                    const uint32_t ke = (kb + p.KC < p.Kt) ? kb + p.KC : p.Kt;
                    mbar_wait(tmem_empty, acc_ph ^ 1);
                    tc_fence_after();
                    for (uint32_t kt = kb; kt < ke; ++kt) {
                        mbar_wait(&full[st], ph);
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
                                const uint32_t d = tmem + s * W;
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
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> fold mod q -> Morton stores
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;
        const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
        uint32_t acc_ph = 0;
        for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            uint32_t m, n;
            tile_coords(tile, p.Mt, p.Nt, m, n);
            const uint64_t gi = (uint64_t)m * kBM + row;
            const bool row_ok = gi < p.rows;
            const uint64_t rbase = row_ok ? __ldg(p.out_rowoff + gi) : 0;
            for (uint32_t c = 0; c < nchunks; ++c) {
                const bool overwrite = (c == 0) && (p.mode == 2);
                mbar_wait(tmem_full, acc_ph);
                tc_fence_after();
#pragma unroll 1
                for (int j0 = 0; j0 < W; j0 += 16) {
                    const uint64_t gj0 = (uint64_t)n * W + j0;
                    if (gj0 >= p.cols) break;  // warp-uniform
                    const int nvalid = (p.cols - gj0) >= 16 ? 16 : (int)(p.cols - gj0);
                    int32_t acc[Cfg::CLASSES][16];
#pragma unroll
                    for (int k = 0; k < Cfg::CLASSES; ++k)
                        tmem_ld16(tmem + lane_base + k * W + j0, acc[k]);
                    tmem_wait_ld();
                    uint32_t res[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        int64_t lo = 0, hi = 0;
#pragma unroll
                        for (int k = 0; k < Cfg::CLASSES; ++k) {
                            if (k < 4) lo += (int64_t)acc[k][j] << (8 * k);
                            else hi += (int64_t)acc[k][j] << (8 * (k - 4));
                        }
                        uint32_t r = red_signed(lo, p);
                        if (Cfg::CLASSES > 4) {
                            uint32_t h = mulmod(red_signed(hi, p), p.w32, p);
                            r += h;
                            r = r >= p.q ? r - p.q : r;
                        }
                        res[j] = r;
                    }
                    const uint64_t c0 = __ldg(p.out_coloff + gj0);
                    bool vec = p.vec_ok && nvalid == 16 && (c0 & 3) == 0;
                    if (vec) vec = __ldg(p.out_coloff + gj0 + 15) == c0 + 15;
                    if (row_ok) {
                        if (vec) {
                            uint4* dst = reinterpret_cast<uint4*>(p.out + rbase + c0);
#pragma unroll
                            for (int v4 = 0; v4 < 4; ++v4) {
                                uint4 o = overwrite ? make_uint4(0, 0, 0, 0) : dst[v4];
                                uint32_t* ov = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    uint32_t s = ov[e] + res[4 * v4 + e];
                                    ov[e] = s >= p.q ? s - p.q : s;
                                }
                                dst[v4] = o;
                            }
                        } else {
                            for (int j = 0; j < nvalid; ++j) {
                                uint32_t* a = p.out + rbase + __ldg(p.out_coloff + gj0 + j);
                                uint32_t s = (overwrite ? 0u : *a) + res[j];
                                *a = s >= p.q ? s - p.q : s;
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(tmem_empty);
                acc_ph ^= 1;
            }
        }
    }

    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int L>
int configure_gemm_t() {
    return (int)cudaFuncSetAttribute(k_gemm<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     GemmCfg<L>::SMEM);
}

// Writes `value` into every cell of a view (SET with an empty inner dimension).
__global__ void k_fill_view(uint32_t* __restrict__ out, const uint64_t* __restrict__ rowoff,
                            const uint64_t* __restrict__ coloff, uint64_t rows, uint64_t cols,
                            uint32_t value) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < rows * cols;
         x += (uint64_t)gridDim.x * blockDim.x)
        out[rowoff[x / cols] + coloff[x % cols]] = value;
}

template <int L>
int launch_gemm_t(const GemmParams& p, int num_sms, cudaStream_t s) {
    using Cfg = GemmCfg<L>;
    const uint32_t tiles = p.Mt * p.Nt;
    const int grid = (int)(tiles < (uint32_t)num_sms ? tiles : (uint32_t)num_sms);
    k_gemm<L><<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(p);
    return (int)cudaGetLastError();
}

template <int L>
int launch_pack_t(int trans, const uint32_t* src, const uint64_t* rowoff, const uint64_t* coloff,
                  uint64_t R, uint64_t K, uint32_t rpt, uint32_t Rtiles, uint32_t Kt, int8_t* dst,
                  DigitParams dp, cudaStream_t s) {
    const uint64_t blocks = (uint64_t)Rtiles * (rpt / kPackRows) * Kt;
    if (trans)
        k_pack<L, true><<<(unsigned)blocks, 256, 0, s>>>(src, rowoff, coloff, R, K, rpt, Kt, dst, dp);
    else
        k_pack<L, false><<<(unsigned)blocks, 256, 0, s>>>(src, rowoff, coloff, R, K, rpt, Kt, dst, dp);
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

int launch_rm_to_mh(const uint32_t* rm, uint32_t* mh, uint64_t n, TileGeom g, uint32_t q,
                    int* bad_flag, void* stream) {
    k_rm_to_mh<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(rm, mh, n, g, q, bad_flag);
    return (int)cudaGetLastError();
}

int launch_mh_to_rm(const uint32_t* mh, uint32_t* rm, uint64_t n, TileGeom g, void* stream) {
    k_mh_to_rm<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(mh, rm, n, g);
    return (int)cudaGetLastError();
}

int launch_pack(int L, int trans, const uint32_t* src, const uint64_t* rowoff,
                const uint64_t* coloff, uint64_t R, uint64_t K, uint32_t rpt, uint32_t Rtiles,
                uint32_t Kt, int8_t* dst, DigitParams dp, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (L) {
        case 1: return launch_pack_t<1>(trans, src, rowoff, coloff, R, K, rpt, Rtiles, Kt, dst, dp, s);
        case 2: return launch_pack_t<2>(trans, src, rowoff, coloff, R, K, rpt, Rtiles, Kt, dst, dp, s);
        case 3: return launch_pack_t<3>(trans, src, rowoff, coloff, R, K, rpt, Rtiles, Kt, dst, dp, s);
        case 4: return launch_pack_t<4>(trans, src, rowoff, coloff, R, K, rpt, Rtiles, Kt, dst, dp, s);
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
    int e = configure_gemm_t<1>();
    if (!e) e = configure_gemm_t<2>();
    if (!e) e = configure_gemm_t<3>();
    if (!e) e = configure_gemm_t<4>();
    return e;
}

int launch_fill_view(uint32_t* out, const uint64_t* rowoff, const uint64_t* coloff, uint64_t rows,
                     uint64_t cols, uint32_t value, void* stream) {
    if (rows == 0 || cols == 0) return 0;
    const uint64_t total = rows * cols;
    const unsigned blocks = (unsigned)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    k_fill_view<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, rowoff, coloff, rows, cols, value);
    return (int)cudaGetLastError();
}

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

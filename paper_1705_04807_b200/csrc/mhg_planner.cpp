// mhg_planner.cpp -- see mhg_planner.hpp.
#include "mhg_planner.hpp"

#include <algorithm>
#include <array>
#include <map>
#include <utility>
#include <vector>

namespace mhg {

bool layout_ok(uint64_t n, uint64_t t) {
    if (n == 0 || t == 0 || n >= (uint64_t(1) << 32)) return false;
    if (n % t != 0) return false;
    const uint64_t g = n / t;
    return (g & (g - 1)) == 0;
}

uint64_t dilate(uint64_t x) {  // interleave zeros: bit b -> bit 2b (low 32 bits)
    x &= 0xffffffffull;
    x = (x | (x << 16)) & 0x0000ffff0000ffffull;
    x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
    x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

uint64_t undilate(uint64_t x) {
    x &= 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
    x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
    x = (x | (x >> 16)) & 0x00000000ffffffffull;
    return x;
}

uint64_t encode(uint64_t t, uint64_t i, uint64_t j) {
    return ((dilate(i / t) << 1) | dilate(j / t)) * t * t + (i % t) * t + (j % t);
}

uint64_t extract_i(uint64_t t, uint64_t z) { return undilate((z / (t * t)) >> 1) * t + (z % (t * t)) / t; }

uint64_t extract_j(uint64_t t, uint64_t z) { return undilate(z / (t * t)) * t + (z % (t * t)) % t; }

TileGeom tile_geom(uint64_t t) {
    TileGeom g{t, t * t, -1};
    if ((t & (t - 1)) == 0) {
        int s = 0;
        while ((uint64_t(1) << s) < t) ++s;
        g.shift = s;
    }
    return g;
}

bool is_prime(uint32_t x) {
    if (x < 2) return false;
    if (x % 2 == 0) return x == 2;
    for (uint64_t d = 3; d * d <= x; d += 2)
        if (x % d == 0) return false;
    return true;
}

// ------------------------------------------------------------------ limbs
LimbParams limb_params(uint32_t q) {
    LimbParams lp{};
    uint32_t L = 1;
    while ((uint64_t)q > (uint64_t(1) << (8 * L))) ++L;  // q <= 256^L
    lp.L = L;
    uint64_t R = 0;  // (256^(L-1) - 1) / 255 : weight sum of the lower digits
    for (uint32_t s = 0; s + 1 < L; ++s) R = R * 256 + 1;
    const uint64_t hmax = 127 * (R * 256 + 1);  // 127 (256^L - 1) / 255
    const uint64_t half = (q - 1) / 2;
    lp.H = (uint32_t)std::min<uint64_t>(half, hmax);
    const int64_t lo = (int64_t)lp.H + 1 - (int64_t)q, hi = (int64_t)lp.H;
    const uint64_t maxabs = (uint64_t)std::max<int64_t>(-lo, hi);
    uint64_t base_top = 1;
    for (uint32_t s = 0; s + 1 < L; ++s) base_top *= 256;
    for (uint32_t s = 0; s < 4; ++s) lp.bound[s] = 0;
    for (uint32_t s = 0; s + 1 < L; ++s) lp.bound[s] = 128;
    lp.bound[L - 1] = (uint32_t)std::min<uint64_t>(128, (maxabs + 128 * R) / base_top);
    uint64_t worst = 1;
    for (uint32_t c = 0; c + 1 < 2 * L; ++c) {
        uint64_t sum = 0;
        for (uint32_t s = 0; s < L; ++s)
            if (c >= s && c - s < L) sum += (uint64_t)lp.bound[s] * lp.bound[c - s];
        worst = std::max(worst, sum);
    }
    // 2^17 of headroom keeps every class sum plus a q-multiple bias inside
    // 32 bits for the epilogue's 32-bit fold
    lp.k_max = ((uint64_t(1) << 31) - (uint64_t(1) << 17)) / worst;
    return lp;
}

// ------------------------------------------------------- closed-form Counters
uint64_t axis_segments(uint64_t off1, uint64_t off2, uint64_t len, uint64_t S) {
    if (len == 0) return 0;
    const uint64_t c1 = (off1 + len - 1) / S - off1 / S;
    const uint64_t c2 = (off2 + len - 1) / S - off2 / S;
    const bool same_phase = (off1 % S) == (off2 % S);
    return 1 + c1 + c2 - (same_phase ? c1 : 0);
}

namespace {

struct LeafAxis {
    uint64_t count = 0, min_len = 0;
    bool any_long = false;  // some leaf piece spans >= 2 cells
};

// Leaf-level pieces of one axis (cut at tile boundaries of either view).
LeafAxis leaf_axis(uint64_t off1, uint64_t off2, uint64_t len, uint64_t t) {
    LeafAxis a;
    if (len == 0) return a;
    std::vector<uint64_t> cuts;
    for (uint64_t off : {off1, off2}) {
        uint64_t x = t - off % t;  // first x >= 1 with (off + x) % t == 0
        for (; x < len; x += t) cuts.push_back(x);
    }
    cuts.push_back(0);
    cuts.push_back(len);
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    a.count = cuts.size() - 1;
    a.min_len = len;
    for (size_t s = 1; s < cuts.size(); ++s) {
        const uint64_t piece = cuts[s] - cuts[s - 1];
        a.min_len = std::min(a.min_len, piece);
        a.any_long = a.any_long || piece >= 2;
    }
    return a;
}

}  // namespace

Counters oblivious_counters(uint64_t n, uint64_t t, const Rect& out, const Rect& lhs,
                            const Rect& rhs) {
    Counters c;
    const uint64_t r = out.rows, cc = out.cols, k = lhs.cols;
    if (r == 0 || cc == 0 || k == 0) return c;  // multiply.hpp:303
    c.scalar_macs = r * k * cc;                 // multiply.hpp:171
    // recursion nodes: depth d = 0..m, block side S = n >> d (multiply.hpp:233-263)
    for (uint64_t S = n; S >= t; S /= 2) {
        c.recursive_calls += axis_segments(out.i, lhs.i, r, S) * axis_segments(lhs.j, rhs.i, k, S) *
                             axis_segments(out.j, rhs.j, cc, S);
        if (S == t) break;
    }
    const LeafAxis X = leaf_axis(out.i, lhs.i, r, t);
    const LeafAxis Z = leaf_axis(lhs.j, rhs.i, k, t);
    const LeafAxis Y = leaf_axis(out.j, rhs.j, cc, t);
    c.base_case_calls = X.count * Z.count * Y.count;
    // JumpTracker (multiply.hpp:80-90) over base_case_mm's walks (:153-170):
    //  out: +1 along a row, t - cols + 1 to the next row;
    //  lhs: +1 along a row, t - inner + 1 to the next row;
    //  rhs: +t down a column, +1 across columns only when inner == 1.
    uint64_t jump = 0;
    if (X.any_long) jump = std::max({jump, t - Y.min_len + 1, t - Z.min_len + 1});
    if (Y.any_long || Z.any_long) jump = std::max<uint64_t>(jump, 1);
    if (Z.any_long) jump = std::max(jump, t);
    c.max_consecutive_jump = jump;
    c.encode_calls = 0;  // contained leaves use offset arithmetic only
    return c;
}

// ------------------------------------ mm_naive / mm_default Counters (closed form)
namespace {

using i128 = __int128;
using Segs = std::vector<std::pair<uint64_t, uint64_t>>;  // (offset in the view, length)
constexpr i128 kNone = -((i128)1 << 100);

// encode = rowpart(i) + colpart(j) (layout.hpp:80-85; the two parts own disjoint bits)
i128 rowpart(uint64_t t, uint64_t i) { return (i128)((dilate(i / t) << 1) * t * t + (i % t) * t); }
i128 colpart(uint64_t t, uint64_t j) { return (i128)(dilate(j / t) * t * t + j % t); }

// dilate(b + 1) - dilate(b) = (2 * 4^m + 1) / 3 for b with m trailing ones: the b in
// [lo, hi] with the most trailing ones has the largest step.
uint64_t most_trailing_ones(uint64_t lo, uint64_t hi) {
    uint64_t best = lo;
    for (int m = 1; m < 63; ++m) {
        const uint64_t want = (uint64_t(1) << m) - 1;
        const uint64_t b = lo + ((want - (lo & want)) & want);  // least b >= lo, b % 2^m == 2^m - 1
        if (b < lo || b > hi) break;
        best = b;
    }
    return best;
}

// max over x in [x0, x0 + len - 2] of part(x + 1) - part(x), len >= 2.  A step across a
// tile boundary (x + 1 == 0 mod t) is never smaller than a step inside a tile (colpart:
// >= t^2 - t + 1 vs 1; rowpart: >= t^2 + t vs t), so the boundary with the most trailing
// ones in its tile index wins when the range holds a boundary.
template <typename Part>
i128 max_step(uint64_t t, uint64_t x0, uint64_t len, Part part) {
    const uint64_t x1 = x0 + len - 2;
    const uint64_t fb = ((x0 + t) / t) * t - 1;  // least x >= x0 with (x + 1) % t == 0
    if (fb <= x1) {
        const uint64_t b = most_trailing_ones(fb / t, (x1 + 1) / t - 1);
        const uint64_t x = b * t + t - 1;
        return part(x + 1) - part(x);
    }
    return part(x0 + 1) - part(x0);  // inside one tile
}

void halving_segments(uint64_t off, uint64_t d, uint64_t t, Segs& out) {
    if (d <= t) {
        out.emplace_back(off, d);
        return;
    }
    const uint64_t d1 = (d + 1) / 2;  // multiply.hpp:212-214
    halving_segments(off, d1, t, out);
    halving_segments(off + d1, d - d1, t, out);
}

void raise(uint64_t& best, i128 gap) {
    if (gap > 0 && gap > (i128)best) best = (uint64_t)gap;
}

// The largest forward gap of JumpTracker (multiply.hpp:80-90) over kernel_encoded calls
// (:104-129) on every leaf (row segment x inner segment x column segment); each call has
// fresh trackers, one per operand, fed in loop order x, y, z.  Every gap kind is a sum
// of independent terms of at most two segment lists, so the maximum separates.
uint64_t encoded_max_jump(const Kernel3& g, const Segs& R, const Segs& K, const Segs& C) {
    auto rowp = [](uint64_t t) { return [t](uint64_t i) { return rowpart(t, i); }; };
    auto colp = [](uint64_t t) { return [t](uint64_t j) { return colpart(t, j); }; };
    // largest step inside any segment of length >= 2 (kNone if none)
    auto steps = [](const Segs& S, uint64_t base, uint64_t t, auto part) {
        i128 m = kNone;
        for (const auto& s : S)
            if (s.second >= 2) m = std::max(m, max_step(t, base + s.first, s.second, part));
        return m;
    };
    // largest part(first) - part(last) of a segment: the backward jump of a rescan
    auto spans = [](const Segs& S, uint64_t base, auto part) {
        i128 m = kNone;
        for (const auto& s : S) m = std::max(m, part(base + s.first) - part(base + s.first + s.second - 1));
        return m;
    };
    uint64_t best = 0;
    const Geo &A = g.out, &B = g.lhs, &Cg = g.rhs;
    // out (ia + x, ja + y): colpart steps along a row; next row: rowpart step + span back
    raise(best, steps(C, A.j, A.t, colp(A.t)));
    if (const i128 rs = steps(R, A.i, A.t, rowp(A.t)); rs > kNone) raise(best, rs + spans(C, A.j, colp(A.t)));
    // lhs (ib + x, jb + z): colpart steps along z; a new y rescans the row (backward);
    // a new x: rowpart step + span back
    raise(best, steps(K, B.j, B.t, colp(B.t)));
    if (const i128 rs = steps(R, B.i, B.t, rowp(B.t)); rs > kNone) raise(best, rs + spans(K, B.j, colp(B.t)));
    // rhs (ic + z, jc + y): rowpart steps along z; a new y: span back + colpart step; a new
    // x restarts at (ic, jc) (backward)
    raise(best, steps(K, Cg.i, Cg.t, rowp(Cg.t)));
    if (const i128 cs = steps(C, Cg.j, Cg.t, colp(Cg.t)); cs > kNone) raise(best, cs + spans(K, Cg.i, rowp(Cg.t)));
    return best;
}

}  // namespace

Counters naive_counters(const Kernel3& g) {
    Counters c;
    const uint64_t r = g.rows, k = g.inner, cc = g.cols;
    if (r == 0 || cc == 0 || k == 0) return c;  // multiply.hpp:272
    c.recursive_calls = 1;
    c.base_case_calls = 1;
    c.scalar_macs = r * k * cc;
    c.encode_calls = r * cc * (2 * k + 1);
    c.max_consecutive_jump = encoded_max_jump(g, {{0, r}}, {{0, k}}, {{0, cc}});
    return c;
}

Counters default_counters(const Kernel3& g) {
    Counters c;
    const uint64_t r = g.rows, k = g.inner, cc = g.cols;
    if (r == 0 || cc == 0 || k == 0) return c;  // multiply.hpp:286
    const uint64_t t = g.out.t;                 // the output layout's tile side (:288)
    Segs R, K, C;
    halving_segments(0, r, t, R);
    halving_segments(0, k, t, K);
    halving_segments(0, cc, t, C);
    c.base_case_calls = R.size() * K.size() * C.size();
    c.scalar_macs = r * k * cc;
    c.encode_calls = r * cc * K.size() + 2 * r * k * cc;
    // nodes: each dimension above t is halved at every level (multiply.hpp:204-229); the
    // shapes at one depth take at most two values per dimension, so memoise by shape
    struct Walk {
        uint64_t t;
        std::map<std::array<uint64_t, 3>, uint64_t> memo;
        uint64_t nodes(uint64_t a, uint64_t b, uint64_t d) {
            if (a <= t && b <= t && d <= t) return 1;
            const std::array<uint64_t, 3> key{a, b, d};
            if (auto it = memo.find(key); it != memo.end()) return it->second;
            auto halves = [&](uint64_t x) {
                return x > t ? std::array<uint64_t, 2>{(x + 1) / 2, x / 2} : std::array<uint64_t, 2>{x, 0};
            };
            uint64_t acc = 1;
            for (uint64_t aa : halves(a))
                for (uint64_t dd : halves(d))
                    for (uint64_t bb : halves(b))
                        if (aa && bb && dd) acc += nodes(aa, bb, dd);
            memo[key] = acc;
            return acc;
        }
    } walk{t, {}};
    c.recursive_calls = walk.nodes(r, k, cc);
    c.max_consecutive_jump = encoded_max_jump(g, R, K, C);
    return c;
}

// -------------------------------------------------------------- task grid
int fold_level(uint32_t q, uint64_t k_chunk) {
    if (q < 2 || q > 65536) return 3;
    const uint64_t w16 = (uint64_t(1) << 16) % q;
    if (w16 >= 256) return 3;
    // |a0|, |a2| <= 2^14 k; |a1| <= 2^15 k, so |a1 >> 8| <= 2^7 k; 0 <= a1l <= 255;
    // cur < q before the chunk
    const uint64_t lim = (uint64_t(1) << 31) - (uint64_t(1) << 17);
    const uint64_t common = (uint64_t)(q - 1) + (uint64_t(1) << 14) * k_chunk + 255 * 256 +
                            w16 * ((uint64_t(1) << 7) * k_chunk);
    if (common + w16 * ((uint64_t(1) << 14) * k_chunk) <= lim) return 1;
    if (common + w16 * (uint64_t)(q - 1) <= lim) return 2;
    return 3;
}

int fold_level_u8(uint32_t q, uint64_t k_chunk) {
    if (q < 2 || q > 65536) return 3;
    const uint64_t w16 = (uint64_t(1) << 16) % q;
    if (w16 >= 256) return 3;
    // unsigned digits, no bias (every class sum >= 0): a0, a2 <= 255^2 k, a1 <= 2 * 255^2 k
    // (< 2^31); both layouts of the partial fold sum cur + a0 + 256 a1l + w16 a1h + w16 t
    // with t = a2 (level 1) or t = a2 mod q (level 2) in uint32 before one reduction
    const uint64_t lim = (uint64_t(1) << 32) - (uint64_t(1) << 17);
    const uint64_t a0 = 65025 * k_chunk, a1h = (130050 * k_chunk) >> 8, a2 = 65025 * k_chunk;
    const uint64_t common = (uint64_t)(q - 1) + a0 + 255 * 256 + w16 * a1h;
    if (common + w16 * a2 <= lim) return 1;
    if (common + w16 * (uint64_t)(q - 1) <= lim) return 2;
    return 3;
}

GemmGeometry gemm_geometry(uint32_t q, uint64_t rows, uint64_t inner, uint64_t cols) {
    const LimbParams lp = limb_params(q);
    GemmGeometry g{};
    g.L = lp.L;
    g.W = (uint32_t)tile_width((int)lp.L);
    g.Mt = (uint32_t)((rows + kBM - 1) / kBM);
    // Kernel: single CTA for L <= 2 -- under the B200's 1 kW cap it sustains higher
    // clocks than the CTA-pair kernel for the same work (profiles/ab_gemm.py,
    // r01_ab_pair_vs_1cta.txt).  Three- and four-limb primes take the pair: their W = 64
    // tiles halve the 1-CTA kernel's output per B' byte, and the pair's shared B' is
    // faster at every K (L = 3: -7..-13%, L = 4: -2..-4%; profiles/r01_pair_wide_primes.txt).
    // MHG_OPT_GEMM_KERNEL forces one (both are exact for every q).
    const int64_t kernel = option(kOptGemmKernel);
    g.pair = kernel == 0 ? lp.L >= 3 : kernel == 2;
    if (g.pair) g.Mt += g.Mt & 1u;  // pairs take two row tiles
    // Problems of at most half a wave of 128 x 128 tiles (e.g. cfg1, n = 512: 16 tiles) are a
    // single latency chain per CTA (load, MMA, drain, store): 128 x 64 tiles put twice as many
    // SMs on it, each with half the chain (profiles/r02b/README.md).
    g.narrow = !g.pair && lp.L <= 2 && option(kOptGemmKernel) != 1 &&
               (uint64_t)g.Mt * ((cols + 127) / 128) <= 74;
    if (g.narrow) g.W = 64;
    g.Nt = (uint32_t)((cols + g.W - 1) / g.W);
    g.Kt = (uint32_t)((inner + kBK - 1) / kBK);
    g.KC = (uint32_t)std::max<uint64_t>(1, lp.k_max / kBK);
    // Unsigned digits (u8 x u8 MMA; 1-CTA and CTA-pair kernels), the default: every class
    // sum is non-negative, so the int32 accumulators grow monotonically instead of
    // random-walking around 0 -- fewer bit toggles, less power -- and the epilogue needs no
    // bias (lean fold levels from fold_level_u8).  Measured faster at every K
    // (profiles/r01_unsigned_digits.txt).  The middle class sums L products of up to
    // 255 * 255 per k, so exact chunks are shorter (16,384 at L = 2 -- the north star's K in one chunk -- vs
    // 65,532 signed).
    // MHG_OPT_DIGITS = 0 selects balanced signed digits.
    g.udig = option(kOptDigits) != 0;
    if (g.udig) {
        const uint64_t kmax_u = ((uint64_t(1) << 31) - (uint64_t(1) << 17)) / ((uint64_t)lp.L * 65025);
        g.KC = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(g.KC, kmax_u / kBK));
    }
    // test hook: a smaller chunk exercises the multi-chunk path on small inputs
    const int64_t cap = option(kOptMaxKChunk);
    if (cap > 0 && (uint64_t)cap < g.KC) g.KC = (uint32_t)cap;
    g.chunks = g.Kt ? (g.Kt + g.KC - 1) / g.KC : 0;
    g.apack_bytes = (uint64_t)g.Mt * kBM * g.Kt * kBK * g.L;
    g.bpack_bytes = (uint64_t)g.Nt * g.W * g.Kt * kBK * g.L;
    return g;
}

// ------------------------------------------------- multi-GPU partition geometry
namespace {
int rank_bits(uint32_t P) {
    if (P == 0 || (P & (P - 1))) return -1;
    int b = 0;
    while ((1u << b) < P) ++b;
    return b;
}
}  // namespace

int dist_block(uint32_t P, uint32_t rank, uint64_t n, uint64_t t, DistBlock& out) {
    const int b = rank_bits(P);
    if (b < 0) return 1;
    if (rank >= P) return 2;
    const uint64_t tiles = n / t;
    if (tiles * tiles < P) return 3;
    const int row_bits = (b + 1) / 2, col_bits = b / 2;
    uint32_t rb = 0, cb = 0;
    for (int k = 0; k < b; ++k) {  // from the most significant bit of rank
        const uint32_t bit = (rank >> (b - 1 - k)) & 1u;
        if (k % 2 == 0) rb = (rb << 1) | bit;
        else cb = (cb << 1) | bit;
    }
    const uint64_t rows = n >> row_bits, cols = n >> col_bits;
    out = DistBlock{rank, rb * rows, cb * cols, rows, cols, rb, cb};
    return 0;
}

uint32_t dist_segment_count(uint32_t P) {
    const int b = rank_bits(P);
    return b < 0 ? 0u : 1u << ((b + 1) / 2);
}

int dist_segment(uint32_t P, uint32_t rank, uint64_t n, uint64_t t, uint32_t index, DistSegment& out) {
    DistBlock blk{};
    if (int e = dist_block(P, rank, n, t, blk)) return e;
    const int b = rank_bits(P);
    const int row_bits = (b + 1) / 2, col_bits = b / 2;
    if (index >= (1u << row_bits)) return 2;
    const uint64_t h = n >> row_bits, w = n >> col_bits;  // band height / width, w in {h, 2h}
    // rank of the block at (row band, column band): interleave their bits back
    auto owner = [&](uint32_t rband, uint32_t cband) {
        uint32_t r = 0;
        for (int k = 0; k < b; ++k) {
            const uint32_t bit = (k % 2 == 0) ? (rband >> (row_bits - 1 - k / 2)) & 1u
                                              : (cband >> (col_bits - 1 - k / 2)) & 1u;
            r = (r << 1) | bit;
        }
        return r;
    };
    const uint64_t per = n * n / P;
    const uint64_t k0 = (uint64_t)index * h;
    const uint32_t a_owner = owner(blk.row_band, (uint32_t)(k0 / w));
    const uint64_t lo = (uint64_t)a_owner * per;
    const uint64_t half = per / (w / h);  // the slice is (w / h) h x h quadrants in Z order
    const uint64_t part = (k0 % w) / h;
    const uint32_t b_owner = owner(index, blk.col_band);
    out = DistSegment{index, k0, k0 + h, a_owner, lo + part * half, lo + (part + 1) * half,
                      b_owner, (uint64_t)b_owner * per, (uint64_t)(b_owner + 1) * per};
    return 0;
}

}  // namespace mhg

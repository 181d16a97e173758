// mhg_planner.hpp -- host-side planner of the Morton-hybrid GF(p) MM path.
//
// The reference reaches its base cases through a recursion on the three
// containers (oblivious_rec, multiply.hpp:232-264; split_sub,
// submatrix.hpp:114-156; compatible_parts, multiply.hpp:177-198).  Its
// decomposition has a closed form (pinned by the reference's own test,
// multiply_test.cpp:79-86 and :252-256): the nodes at recursion depth d are the
// Cartesian product of three 1-D segmentations, each axis cut wherever either
// of the two views sharing it crosses a multiple of the depth-d block side
// n / 2^d.  The planner evaluates that closed form (Counters) and turns the
// problem into a flat grid of aligned tile-block GEMM tasks over packed operands
// -- no device recursion, no index conversion inside the kernels.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "mhg_internal.hpp"

namespace mhg {

// ------------------------------------------------------------ codec (host)
bool layout_ok(uint64_t n, uint64_t t);  // Layout(n, t) preconditions, layout.hpp:50-56
uint64_t dilate(uint64_t x);
uint64_t undilate(uint64_t x);
uint64_t encode(uint64_t t, uint64_t i, uint64_t j);
uint64_t extract_i(uint64_t t, uint64_t z);
uint64_t extract_j(uint64_t t, uint64_t z);
TileGeom tile_geom(uint64_t t);
bool is_prime(uint32_t q);

// ------------------------------------------------------ closed-form Counters
struct Rect {
    uint64_t i, j, rows, cols;  // container coordinates of the view
};

struct Counters {
    uint64_t base_case_calls = 0, scalar_macs = 0, encode_calls = 0, recursive_calls = 0,
             max_consecutive_jump = 0;
};

// Number of pieces of [0, len) cut where (off1 + x) % S == 0 or (off2 + x) % S == 0.
uint64_t axis_segments(uint64_t off1, uint64_t off2, uint64_t len, uint64_t S);

// Counters of mm_oblivious for out(r x c) += lhs(r x k) * rhs(k x c).
Counters oblivious_counters(uint64_t n, uint64_t t, const Rect& out, const Rect& lhs,
                            const Rect& rhs);

// Geometry of one view for the encode-addressed kernels, whose three containers may
// have different layouts: tile side t and the view's first cell (i, j).
struct Geo {
    uint64_t n, t, i, j;
};
struct Kernel3 {
    Geo out, lhs, rhs;
    uint64_t rows, inner, cols;
};
// Counters of mm_naive (multiply.hpp:269-278) and mm_default (:283-291), closed form
// (including max_consecutive_jump of their encode-addressed walks).
Counters naive_counters(const Kernel3& g);
Counters default_counters(const Kernel3& g);

// -------------------------------------------------------------- task grid
struct GemmGeometry {
    bool pair;            // CTA-pair kernel (k_gemm2); Mt is then even
    bool narrow;          // 128 x 64 tiles for a problem of <= 74 128 x 128 tiles (1-2 limbs)
    bool udig;            // unsigned u8 digits (MHG_OPT_DIGITS = 1, the default)
    uint32_t L, W;        // limbs, output tile width
    uint32_t Mt, Nt, Kt;  // tiles along rows / cols / inner (128-byte K slices)
    uint32_t KC;          // K slices per exact int32 chunk
    uint32_t chunks;
    uint64_t apack_bytes, bpack_bytes;
};

GemmGeometry gemm_geometry(uint32_t q, uint64_t rows, uint64_t inner, uint64_t cols);

// Cheapest exact fold level of the lean L = 2 epilogue (GemmParams::fold) for
// chunks of k_chunk inner products (w16 = 2^16 mod q < 256; 3 otherwise):
//   1 if  cur + a0 + 256 a1l + w16 (a1h + a2)  stays within 2^31 - 2^17,
//   2 if  cur + a0 + 256 a1l + w16 a1h + w16 (a2 mod q)  does, else 3.
int fold_level(uint32_t q, uint64_t k_chunk);
// The same for unsigned (u8) digits: class sums are non-negative, so the kernel runs
// without the q-multiple bias (GemmParams::bias32 = 0) and the levels test uint32 range.
int fold_level_u8(uint32_t q, uint64_t k_chunk);

// ------------------------------------------------- multi-GPU partition geometry
// C-stationary partition by top-level Morton blocks: with P = 2^b ranks,
// rank r owns the r-th contiguous 1/P slice of every container's flat store -- a
// rectangle, because the Z order visits quadrants NW, NE, SW, SE at every scale
// (layout.hpp:42-48): the bits of r, most significant first, alternate row-half /
// column-half choices.  Rank r updates C[R_r, C_r]; K is cut at row-band boundaries
// into segments whose A part is a contiguous flat range of ONE row-group member's
// slice and whose B part is the whole slice of ONE column-group member.
struct DistBlock {
    uint32_t rank;
    uint64_t i0, j0, rows, cols;
    uint32_t row_band, col_band;
};
struct DistSegment {
    uint32_t index;
    uint64_t k0, k1;
    uint32_t a_owner;
    uint64_t a_begin, a_end;  // flat cell range of A[R_r, k0:k1] (in a_owner's slice)
    uint32_t b_owner;
    uint64_t b_begin, b_end;  // flat cell range of B[k0:k1, C_r] (b_owner's whole slice)
};
// 0 on success; 1 = P not a power of two, 2 = rank out of range, 3 = fewer tiles than ranks
int dist_block(uint32_t P, uint32_t rank, uint64_t n, uint64_t t, DistBlock& out);
uint32_t dist_segment_count(uint32_t P);  // row bands = K segments per rank
int dist_segment(uint32_t P, uint32_t rank, uint64_t n, uint64_t t, uint32_t index, DistSegment& out);

}  // namespace mhg

/*
 * mh_oracle.h -- CPU restatement of the reference's Morton-hybrid GF(p) MM path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (libmhg.so) never links or calls it.
 *
 * Everything here is plain C11 restating, function by function, what the
 * reference computes (citations are paths under the reference's proj/):
 *   - seeded generator      include/mh/bench.hpp:44-52   (mt19937_64 + 128-bit below)
 *   - instance draws        include/mh/bench.hpp:71-110  (gen_problem)
 *   - Morton-hybrid codec   include/mh/layout.hpp:15-99  (dilate / encode / extract)
 *   - field arithmetic      include/mh/field.hpp:43-55   (canonical add / mul mod q)
 *   - descriptor predicates include/mh/submatrix.hpp:43-156
 *   - mm_oblivious          include/mh/multiply.hpp:232-264, 297-308 (recursion,
 *                           Counters), base_case_mm :136-172, compatible_parts :177-198
 *   - dense oracle          tests/support/oracles.hpp:46-58 (mat_mul_accumulate)
 * plus two size-independent checkers used at full benchmark sizes:
 *   - Freivalds' identity   (C_new - C_old) r == s * A (B r)   mod q
 *   - sampled-tile dense recompute of chosen output rectangles.
 *
 * Pinned against the reference's golden vectors (tests/golden/, tests/test_oracle_*.py)
 * and against the reference library itself compiled from /root/reference
 * (oracle/ref_shim.cpp -> oracle/_ref/libmhref.so).
 */
#ifndef MH_ORACLE_H
#define MH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference's exception classes */
enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_OUT_OF_RANGE = 2, ORC_LOGIC_ERROR = 3 };

/* ---- generator (bench.hpp:44-52) ---- */
typedef struct {
    uint64_t state[312];
    int pos;
} orc_rng;

void orc_rng_seed(orc_rng *g, uint64_t seed);
uint64_t orc_rng_next(orc_rng *g);
uint64_t orc_rng_below(orc_rng *g, uint64_t k);
orc_rng *orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng *g);
/* cells[z] = below(q) for z = 0..count-1 (flat order, bench.hpp:101-103) */
void orc_fill_below(orc_rng *g, uint32_t *cells, uint64_t count, uint32_t q);

/* ---- field (field.hpp:10-55) ---- */
int orc_is_prime(uint32_t x);
uint32_t orc_add(uint32_t a, uint32_t b, uint32_t q);
uint32_t orc_mul(uint32_t a, uint32_t b, uint32_t q);

/* ---- codec (layout.hpp) ---- */
int orc_layout_check(uint64_t n, uint64_t t); /* 0 or ORC_INVALID_ARGUMENT */
uint64_t orc_dilate(uint64_t x);
uint64_t orc_undilate(uint64_t x);
uint64_t orc_encode(uint64_t n, uint64_t t, uint64_t i, uint64_t j);
uint64_t orc_extract_i(uint64_t n, uint64_t t, uint64_t z);
uint64_t orc_extract_j(uint64_t n, uint64_t t, uint64_t z);

/* ---- instance draw (bench.hpp:71-110) ----
 * desc[0] aligned_draw, [1..3] out origin/rows/cols, [4..6] lhs, [7..9] rhs.
 * out/lhs/rhs receive n*n cells each (drawn in that order). */
int orc_gen_problem(orc_rng *g, uint64_t n, uint64_t t, uint32_t q, uint32_t *out,
                    uint32_t *lhs, uint32_t *rhs, uint64_t desc[10]);

/* ---- Counters (multiply.hpp:39-45) ---- */
typedef struct {
    uint64_t base_case_calls;
    uint64_t scalar_macs;
    uint64_t encode_calls;
    uint64_t recursive_calls;
    uint64_t max_consecutive_jump;
} orc_counters;

/* View triple inside three n x n containers sharing (n, t, q). */
typedef struct {
    uint64_t n, t;
    uint32_t q;
    uint32_t *out;        /* updated in place */
    const uint32_t *lhs;
    const uint32_t *rhs;
    uint64_t out_origin, lhs_origin, rhs_origin; /* flat Morton-hybrid index of first entry */
    uint64_t rows, inner, cols;
} orc_problem;

/* Faithful restatement of mm_oblivious: out += lhs * rhs with the aligned
 * container recursion and contained base cases; fills Counters exactly as the
 * reference does.  Intended for small n (it is a scalar triple loop). */
int orc_mm_oblivious(const orc_problem *p, orc_counters *ctr);

/* Dense checker (oracles.hpp:46-58 semantics, blocked, delayed reduction,
 * `threads` POSIX threads over disjoint output rows).
 * op: 0 out += lhs*rhs, 1 out -= lhs*rhs, 2 out = lhs*rhs (view only). */
int orc_mm_dense(const orc_problem *p, int op, int threads);

/* Dense recompute of an output sub-rectangle [r0, r0+nr) x [c0, c0+nc) of the
 * view, written to dst (row-major nr x nc) given the ORIGINAL out cells. */
int orc_mm_dense_block(const orc_problem *p, int op, uint64_t r0, uint64_t nr, uint64_t c0,
                       uint64_t nc, uint32_t *dst, int threads);

/* Freivalds: for `rounds` random vectors v (seeded), checks
 *   new_out_view * v == old_out_view * v + s * lhs * (rhs * v)   (mod q),
 * s = +1 (op 0), -1 (op 1); op 2 ignores old.  Returns 1 if all rounds pass,
 * 0 on mismatch, negative on error.  new_out is the updated container. */
int orc_freivalds(const orc_problem *p_old, const uint32_t *new_out, int op, int rounds,
                  uint64_t seed, int threads);

/* Row-major <-> Morton-hybrid permutations (matrix.hpp:44-67). */
int orc_rowmajor_to_mh(uint64_t n, uint64_t t, const uint32_t *rows, uint32_t *cells);
int orc_mh_to_rowmajor(uint64_t n, uint64_t t, const uint32_t *cells, uint32_t *rows);

#ifdef __cplusplus
}
#endif

#endif

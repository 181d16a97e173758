/*
 * mh_oracle.c -- CPU restatement of the reference path (see mh_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: the checker the GPU path is compared against.
 * Never linked into libmhg.so; never on the product path.
 */
#include "mh_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ generator
 * std::mt19937_64 (Matsumoto-Nishimura 64-bit Mersenne twister, the engine the
 * reference seeds in bench.hpp:47) restated from its published parameters. */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_rng_seed(orc_rng *g, uint64_t seed) {
    g->state[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        const uint64_t prev = g->state[i - 1];
        g->state[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
    }
    g->pos = MT_N;
}

static void mt_twist(orc_rng *g) {
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t y = (g->state[i] & MT_UPPER) | (g->state[(i + 1) % MT_N] & MT_LOWER);
        uint64_t v = g->state[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
        g->state[i] = v;
    }
    g->pos = 0;
}

uint64_t orc_rng_next(orc_rng *g) {
    if (g->pos >= MT_N) mt_twist(g);
    uint64_t x = g->state[g->pos++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* bench.hpp:49-51: multiply-high mapping of a 64-bit draw onto [0, k). */
uint64_t orc_rng_below(orc_rng *g, uint64_t k) {
    return (uint64_t)(((u128)orc_rng_next(g) * (u128)k) >> 64);
}

orc_rng *orc_rng_new(uint64_t seed) {
    orc_rng *g = (orc_rng *)malloc(sizeof(orc_rng));
    if (g) orc_rng_seed(g, seed);
    return g;
}

void orc_rng_free(orc_rng *g) { free(g); }

void orc_fill_below(orc_rng *g, uint32_t *cells, uint64_t count, uint32_t q) {
    for (uint64_t z = 0; z < count; ++z) cells[z] = (uint32_t)orc_rng_below(g, q);
}

/* ---------------------------------------------------------------------- field */
int orc_is_prime(uint32_t x) { /* field.hpp:10-16 (trial division) */
    if (x < 2) return 0;
    if (x % 2 == 0) return x == 2;
    for (uint64_t d = 3; d * d <= x; d += 2)
        if (x % d == 0) return 0;
    return 1;
}

uint32_t orc_add(uint32_t a, uint32_t b, uint32_t q) { /* field.hpp:43-47 */
    uint32_t s = a + b;
    return s >= q ? s - q : s;
}

uint32_t orc_mul(uint32_t a, uint32_t b, uint32_t q) { /* field.hpp:49-55, canonical result */
    return (uint32_t)(((uint64_t)a * b) % q);
}

/* ---------------------------------------------------------------------- codec */
static int is_pow2(uint64_t v) { return v && !(v & (v - 1)); }

int orc_layout_check(uint64_t n, uint64_t t) { /* layout.hpp:50-62 */
    if (n == 0 || t == 0) return ORC_INVALID_ARGUMENT;
    if (n >= (1ULL << 32)) return ORC_INVALID_ARGUMENT;
    if (n % t != 0 || !is_pow2(n / t)) return ORC_INVALID_ARGUMENT;
    return ORC_OK;
}

uint64_t orc_dilate(uint64_t x) { /* bit k -> bit 2k, layout.hpp:15-23 */
    uint64_t out = 0;
    for (int b = 0; b < 32; ++b) out |= ((x >> b) & 1ULL) << (2 * b);
    return out;
}

uint64_t orc_undilate(uint64_t x) { /* even bits -> packed, layout.hpp:25-33 */
    uint64_t out = 0;
    for (int b = 0; b < 32; ++b) out |= ((x >> (2 * b)) & 1ULL) << b;
    return out;
}

uint64_t orc_encode(uint64_t n, uint64_t t, uint64_t i, uint64_t j) { /* layout.hpp:80-85 */
    (void)n;
    const uint64_t zb = (orc_dilate(i / t) << 1) | orc_dilate(j / t);
    return zb * t * t + (i % t) * t + (j % t);
}

uint64_t orc_extract_i(uint64_t n, uint64_t t, uint64_t z) { /* layout.hpp:88-92 */
    (void)n;
    return orc_undilate((z / (t * t)) >> 1) * t + (z % (t * t)) / t;
}

uint64_t orc_extract_j(uint64_t n, uint64_t t, uint64_t z) { /* layout.hpp:95-99 */
    (void)n;
    return orc_undilate(z / (t * t)) * t + (z % (t * t)) % t;
}

int orc_rowmajor_to_mh(uint64_t n, uint64_t t, const uint32_t *rows, uint32_t *cells) {
    if (orc_layout_check(n, t)) return ORC_INVALID_ARGUMENT;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < n; ++j) cells[orc_encode(n, t, i, j)] = rows[i * n + j];
    return ORC_OK;
}

int orc_mh_to_rowmajor(uint64_t n, uint64_t t, const uint32_t *cells, uint32_t *rows) {
    if (orc_layout_check(n, t)) return ORC_INVALID_ARGUMENT;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < n; ++j) rows[i * n + j] = cells[orc_encode(n, t, i, j)];
    return ORC_OK;
}

/* ------------------------------------------------------------- instance draw */
int orc_gen_problem(orc_rng *g, uint64_t n, uint64_t t, uint32_t q, uint32_t *out,
                    uint32_t *lhs, uint32_t *rhs, uint64_t desc[10]) {
    if (orc_layout_check(n, t) || q < 2 || q >= (1U << 31) || !orc_is_prime(q))
        return ORC_INVALID_ARGUMENT;
    unsigned m = 0;
    while ((t << m) < n) ++m;
    const int aligned = orc_rng_below(g, 8) == 0; /* bench.hpp:65,75 */
    uint64_t r, k, c, ia, ja, ib, jb, ic, jc;
    if (aligned) {
        r = t << orc_rng_below(g, m + 1);
        k = t << orc_rng_below(g, m + 1);
        c = t << orc_rng_below(g, m + 1);
#define CORNER(ext) (t * orc_rng_below(g, (n - (ext)) / t + 1))
        ia = CORNER(r); ja = CORNER(c);
        ib = CORNER(r); jb = CORNER(k);
        ic = CORNER(k); jc = CORNER(c);
#undef CORNER
    } else {
        r = 1 + orc_rng_below(g, n);
        k = 1 + orc_rng_below(g, n);
        c = 1 + orc_rng_below(g, n);
        ia = orc_rng_below(g, n - r + 1); ja = orc_rng_below(g, n - c + 1);
        ib = orc_rng_below(g, n - r + 1); jb = orc_rng_below(g, n - k + 1);
        ic = orc_rng_below(g, n - k + 1); jc = orc_rng_below(g, n - c + 1);
    }
    orc_fill_below(g, out, n * n, q);
    orc_fill_below(g, lhs, n * n, q);
    orc_fill_below(g, rhs, n * n, q);
    desc[0] = (uint64_t)aligned;
    desc[1] = orc_encode(n, t, ia, ja); desc[2] = r; desc[3] = c;
    desc[4] = orc_encode(n, t, ib, jb); desc[5] = r; desc[6] = k;
    desc[7] = orc_encode(n, t, ic, jc); desc[8] = k; desc[9] = c;
    return ORC_OK;
}

/* ------------------------------------------------------- recursion restatement
 * Views are carried as (origin row, origin col, rows, cols) in container
 * coordinates; aligned blocks as (flat origin, element count). */
typedef struct { uint64_t i, j, rows, cols; } rect;
typedef struct { rect v; uint64_t row0, col0; } framed;        /* multiply.hpp:72-76 */
typedef struct { uint64_t origin, elems; } block;              /* submatrix.hpp:22-26 */
typedef struct { int present[4]; rect part[4]; uint64_t rn, cw; } split; /* :35-41 */

typedef struct {
    uint64_t n, t, tile;
    uint32_t q;
    uint32_t *A;             /* out */
    const uint32_t *B, *C;   /* lhs, rhs */
    orc_counters *ctr;
} rec_ctx;

typedef struct { uint64_t last; int armed; } jump_tracker; /* multiply.hpp:80-90 */

static void jt_touch(jump_tracker *jt, uint64_t a, orc_counters *ctr) {
    if (jt->armed && a > jt->last && a - jt->last > ctr->max_consecutive_jump)
        ctr->max_consecutive_jump = a - jt->last;
    jt->last = a;
    jt->armed = 1;
}

static int rect_contained(uint64_t t, const rect *s) { /* submatrix.hpp:87-93 */
    if (s->rows == 0 || s->cols == 0) return 1;
    return s->i / t == (s->i + s->rows - 1) / t && s->j / t == (s->j + s->cols - 1) / t;
}

/* multiply.hpp:136-172: leaf multiply with row-major offsets inside one tile */
static int base_case(rec_ctx *x, const rect *o, const rect *l, const rect *r) {
    if (!rect_contained(x->t, o) || !rect_contained(x->t, l) || !rect_contained(x->t, r))
        return ORC_LOGIC_ERROR;
    if (o->rows != l->rows || o->cols != r->cols || l->cols != r->rows) return ORC_LOGIC_ERROR;
    x->ctr->base_case_calls++;
    const uint64_t t = x->t, n = x->n;
    const uint64_t zo = o->rows ? orc_encode(n, t, o->i, o->j) : 0;
    const uint64_t zl = l->rows ? orc_encode(n, t, l->i, l->j) : 0;
    const uint64_t zr = r->rows ? orc_encode(n, t, r->i, r->j) : 0;
    jump_tracker ja = {0, 0}, jb = {0, 0}, jc = {0, 0};
    for (uint64_t a = 0; a < o->rows; ++a) {
        const uint64_t row_o = zo + a * t, row_l = zl + a * t;
        for (uint64_t b = 0; b < o->cols; ++b) {
            const uint64_t za = row_o + b;
            jt_touch(&ja, za, x->ctr);
            uint32_t acc = x->A[za];
            uint64_t zc = zr + b;
            for (uint64_t z = 0; z < l->cols; ++z) {
                const uint64_t zb = row_l + z;
                jt_touch(&jb, zb, x->ctr);
                jt_touch(&jc, zc, x->ctr);
                acc = orc_add(acc, orc_mul(x->B[zb], x->C[zc], x->q), x->q);
                zc += t;
            }
            x->A[za] = acc;
        }
    }
    x->ctr->scalar_macs += o->rows * o->cols * l->cols;
    return ORC_OK;
}

static uint64_t block_side(const rec_ctx *x, const block *b) { /* submatrix.hpp:54-58 */
    uint64_t ratio = b->elems / x->tile, side = x->t;
    while (ratio > 1) { ratio >>= 2; side <<= 1; }
    return side;
}

/* submatrix.hpp:114-156: carve view s along the quadrant boundaries of b */
static split split_view(const rec_ctx *x, const block *b, const rect *s) {
    split out;
    memset(&out, 0, sizeof out);
    const uint64_t quarter = b->elems / 4;
    const uint64_t last_ne = b->origin + 2 * quarter - 1;
    const uint64_t last_sw = b->origin + 3 * quarter - 1;
    long long rn = (long long)orc_extract_i(x->n, x->t, last_ne) - (long long)s->i + 1;
    long long cw = (long long)orc_extract_j(x->n, x->t, last_sw) - (long long)s->j + 1;
    if (rn < 0) rn = 0;
    if ((uint64_t)rn > s->rows) rn = (long long)s->rows;
    if (cw < 0) cw = 0;
    if ((uint64_t)cw > s->cols) cw = (long long)s->cols;
    out.rn = (uint64_t)rn;
    out.cw = (uint64_t)cw;
    const uint64_t rs = s->rows - out.rn, ce = s->cols - out.cw;
    const uint64_t di[4] = {0, 0, out.rn, out.rn}, dj[4] = {0, out.cw, 0, out.cw};
    const uint64_t nr[4] = {out.rn, out.rn, rs, rs}, nc[4] = {out.cw, ce, out.cw, ce};
    for (int qd = 0; qd < 4; ++qd) {
        if (nr[qd] && nc[qd]) {
            out.present[qd] = 1;
            out.part[qd].i = s->i + di[qd];
            out.part[qd].j = s->j + dj[qd];
            out.part[qd].rows = nr[qd];
            out.part[qd].cols = nc[qd];
        }
    }
    (void)block_side;
    return out;
}

static uint64_t umax(uint64_t a, uint64_t b) { return a > b ? a : b; }
static uint64_t umin(uint64_t a, uint64_t b) { return a < b ? a : b; }

/* multiply.hpp:177-198: intersect the shared row / inner / column ranges */
static int compatible(const framed *pa, const framed *pb, const framed *pc, framed out[3]) {
    const uint64_t xl = umax(pa->row0, pb->row0), xh = umin(pa->row0 + pa->v.rows, pb->row0 + pb->v.rows);
    const uint64_t zl = umax(pb->col0, pc->row0), zh = umin(pb->col0 + pb->v.cols, pc->row0 + pc->v.rows);
    const uint64_t yl = umax(pa->col0, pc->col0), yh = umin(pa->col0 + pa->v.cols, pc->col0 + pc->v.cols);
    if (xh <= xl || zh <= zl || yh <= yl) return 0;
#define CUT(dst, f, rl, rh, cl, ch)                                  \
    do {                                                             \
        (dst).v.i = (f)->v.i + ((rl) - (f)->row0);                   \
        (dst).v.j = (f)->v.j + ((cl) - (f)->col0);                   \
        (dst).v.rows = (rh) - (rl);                                  \
        (dst).v.cols = (ch) - (cl);                                  \
        (dst).row0 = (rl);                                           \
        (dst).col0 = (cl);                                           \
    } while (0)
    CUT(out[0], pa, xl, xh, yl, yh);
    CUT(out[1], pb, xl, xh, zl, zh);
    CUT(out[2], pc, zl, zh, yl, yh);
#undef CUT
    return 1;
}

/* multiply.hpp:232-264: lock-step descent of the three aligned block trees */
static int oblivious_rec(rec_ctx *x, const block *ba, const block *bb, const block *bc,
                         const framed *pa, const framed *pb, const framed *pc) {
    x->ctr->recursive_calls++;
    if (ba->elems == x->tile) return base_case(x, &pa->v, &pb->v, &pc->v);
    const uint64_t quarter = ba->elems / 4;
    const split sa = split_view(x, ba, &pa->v);
    const split sb = split_view(x, bb, &pb->v);
    const split sc = split_view(x, bc, &pc->v);
    for (int ta = 0; ta < 4; ++ta) {
        if (!sa.present[ta]) continue;
        const framed fa = {sa.part[ta], pa->row0 + ((ta & 2) ? sa.rn : 0), pa->col0 + ((ta & 1) ? sa.cw : 0)};
        for (int tb = 0; tb < 4; ++tb) {
            if (!sb.present[tb]) continue;
            const framed fb = {sb.part[tb], pb->row0 + ((tb & 2) ? sb.rn : 0), pb->col0 + ((tb & 1) ? sb.cw : 0)};
            for (int tc = 0; tc < 4; ++tc) {
                if (!sc.present[tc]) continue;
                const framed fc = {sc.part[tc], pc->row0 + ((tc & 2) ? sc.rn : 0), pc->col0 + ((tc & 1) ? sc.cw : 0)};
                framed tr[3];
                if (!compatible(&fa, &fb, &fc, tr)) continue;
                const block ca = {ba->origin + (uint64_t)ta * quarter, quarter};
                const block cb = {bb->origin + (uint64_t)tb * quarter, quarter};
                const block cc = {bc->origin + (uint64_t)tc * quarter, quarter};
                const int st = oblivious_rec(x, &ca, &cb, &cc, &tr[0], &tr[1], &tr[2]);
                if (st) return st;
            }
        }
    }
    return ORC_OK;
}

static int check_view(uint64_t n, uint64_t t, uint64_t origin, uint64_t rows, uint64_t cols) {
    if (origin >= n * n) return ORC_OUT_OF_RANGE; /* submatrix.hpp:43-51 */
    if (orc_extract_i(n, t, origin) + rows > n || orc_extract_j(n, t, origin) + cols > n)
        return ORC_OUT_OF_RANGE;
    return ORC_OK;
}

static int check_problem(const orc_problem *p) {
    if (orc_layout_check(p->n, p->t)) return ORC_INVALID_ARGUMENT;
    int st;
    if ((st = check_view(p->n, p->t, p->out_origin, p->rows, p->cols))) return st;
    if ((st = check_view(p->n, p->t, p->lhs_origin, p->rows, p->inner))) return st;
    if ((st = check_view(p->n, p->t, p->rhs_origin, p->inner, p->cols))) return st;
    if ((const uint32_t *)p->out == p->lhs || (const uint32_t *)p->out == p->rhs || p->lhs == p->rhs)
        return ORC_LOGIC_ERROR;
    return ORC_OK;
}

int orc_mm_oblivious(const orc_problem *p, orc_counters *ctr) {
    memset(ctr, 0, sizeof *ctr);
    int st = check_problem(p);
    if (st) return st;
    if (p->rows == 0 || p->cols == 0 || p->inner == 0) return ORC_OK; /* multiply.hpp:303 */
    rec_ctx x = {p->n, p->t, p->t * p->t, p->q, p->out, p->lhs, p->rhs, ctr};
    const block whole = {0, p->n * p->n};
    const uint64_t n = p->n, t = p->t;
    const framed fa = {{orc_extract_i(n, t, p->out_origin), orc_extract_j(n, t, p->out_origin), p->rows, p->cols}, 0, 0};
    const framed fb = {{orc_extract_i(n, t, p->lhs_origin), orc_extract_j(n, t, p->lhs_origin), p->rows, p->inner}, 0, 0};
    const framed fc = {{orc_extract_i(n, t, p->rhs_origin), orc_extract_j(n, t, p->rhs_origin), p->inner, p->cols}, 0, 0};
    return oblivious_rec(&x, &whole, &whole, &whole, &fa, &fb, &fc);
}

/* ------------------------------------------------------------ dense checkers */
typedef struct {
    uint64_t n, t;
    uint64_t *rowpart; /* size n: Morton offset contribution of absolute row i */
    uint64_t *colpart; /* size n: of absolute column j */
} offsets;

static int offsets_make(offsets *o, uint64_t n, uint64_t t) {
    o->n = n;
    o->t = t;
    o->rowpart = (uint64_t *)malloc(n * sizeof(uint64_t));
    o->colpart = (uint64_t *)malloc(n * sizeof(uint64_t));
    if (!o->rowpart || !o->colpart) return -1;
    for (uint64_t i = 0; i < n; ++i) {
        o->rowpart[i] = (orc_dilate(i / t) << 1) * t * t + (i % t) * t;
        o->colpart[i] = orc_dilate(i / t) * t * t + (i % t);
    }
    return 0;
}

static void offsets_free(offsets *o) {
    free(o->rowpart);
    free(o->colpart);
}

typedef struct {
    const orc_problem *p;
    const offsets *off;
    const uint32_t *lhs_rm; /* rows x inner, row-major, already sign-applied */
    const uint32_t *rhs_cm; /* cols x inner (transposed) */
    uint64_t r0, nr, c0, nc;
    uint32_t *dst;          /* if non-null: write nr x nc block here instead of out */
    int op;
    uint64_t row_begin, row_end; /* thread slice, relative to r0 */
} dense_job;

static uint32_t dot_mod(const uint32_t *a, const uint32_t *b, uint64_t k, uint32_t q) {
    if (q <= 65536u) {
        /* products < 2^32: a u64 sum of fewer than 2^32 of them cannot wrap */
        uint64_t acc = 0;
        for (uint64_t z = 0; z < k; ++z) acc += (uint64_t)a[z] * b[z];
        return (uint32_t)(acc % q);
    }
    /* split a into 16-bit halves: each partial product < 2^47 */
    uint64_t lo = 0, hi = 0;
    uint32_t res = 0;
    const uint32_t w16 = (uint32_t)((1ULL << 16) % q);
    for (uint64_t z0 = 0; z0 < k; z0 += 65536) {
        const uint64_t ze = umin(k, z0 + 65536);
        lo = hi = 0;
        for (uint64_t z = z0; z < ze; ++z) {
            lo += (uint64_t)(a[z] & 0xFFFFu) * b[z];
            hi += (uint64_t)(a[z] >> 16) * b[z];
        }
        const uint64_t part = (lo % q + (hi % q) * w16) % q;
        res = (uint32_t)((res + part) % q);
    }
    return res;
}

static void *dense_worker(void *arg) {
    dense_job *j = (dense_job *)arg;
    const orc_problem *p = j->p;
    const offsets *off = j->off;
    const uint64_t oi = orc_extract_i(p->n, p->t, p->out_origin);
    const uint64_t oj = orc_extract_j(p->n, p->t, p->out_origin);
    for (uint64_t a = j->row_begin; a < j->row_end; ++a) {
        const uint64_t x = j->r0 + a;
        const uint32_t *lrow = j->lhs_rm + x * p->inner;
        for (uint64_t b = 0; b < j->nc; ++b) {
            const uint64_t y = j->c0 + b;
            const uint32_t prod = dot_mod(lrow, j->rhs_cm + y * p->inner, p->inner, p->q);
            const uint64_t z = off->rowpart[oi + x] + off->colpart[oj + y];
            uint32_t v;
            if (j->op == 2) v = prod;
            else v = orc_add(p->out[z], prod, p->q);
            if (j->dst) j->dst[a * j->nc + b] = v;
            else p->out[z] = v;
        }
    }
    return NULL;
}

static int dense_impl(const orc_problem *p, int op, uint64_t r0, uint64_t nr, uint64_t c0,
                      uint64_t nc, uint32_t *dst, int threads) {
    int st = check_problem(p);
    if (st) return st;
    if (op < 0 || op > 2) return ORC_INVALID_ARGUMENT;
    if (r0 + nr > p->rows || c0 + nc > p->cols) return ORC_OUT_OF_RANGE;
    if (nr == 0 || nc == 0) return ORC_OK;
    offsets off;
    if (offsets_make(&off, p->n, p->t)) return -1;
    const uint64_t li = orc_extract_i(p->n, p->t, p->lhs_origin), lj = orc_extract_j(p->n, p->t, p->lhs_origin);
    const uint64_t ri = orc_extract_i(p->n, p->t, p->rhs_origin), rj = orc_extract_j(p->n, p->t, p->rhs_origin);
    const uint64_t k = p->inner;
    /* gather only the lhs rows and rhs columns this block needs */
    uint32_t *lhs_rm = (uint32_t *)malloc((r0 + nr) * (k ? k : 1) * sizeof(uint32_t));
    uint32_t *rhs_cm = (uint32_t *)malloc((c0 + nc) * (k ? k : 1) * sizeof(uint32_t));
    if (!lhs_rm || !rhs_cm) {
        free(lhs_rm); free(rhs_cm); offsets_free(&off);
        return -1;
    }
    for (uint64_t x = r0; x < r0 + nr; ++x)
        for (uint64_t z = 0; z < k; ++z) {
            uint32_t v = p->lhs[off.rowpart[li + x] + off.colpart[lj + z]];
            if (op == 1) v = v ? p->q - v : 0; /* C -= A.B  ==  C += (-A).B */
            lhs_rm[x * k + z] = v;
        }
    for (uint64_t z = 0; z < k; ++z)
        for (uint64_t y = c0; y < c0 + nc; ++y)
            rhs_cm[y * k + z] = p->rhs[off.rowpart[ri + z] + off.colpart[rj + y]];
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > nr) threads = (int)nr;
    pthread_t tid[256];
    dense_job jobs[256];
    if (threads > 256) threads = 256;
    for (int w = 0; w < threads; ++w) {
        dense_job *jb = &jobs[w];
        jb->p = p; jb->off = &off; jb->lhs_rm = lhs_rm; jb->rhs_cm = rhs_cm;
        jb->r0 = r0; jb->nr = nr; jb->c0 = c0; jb->nc = nc; jb->dst = dst; jb->op = op;
        jb->row_begin = nr * (uint64_t)w / (uint64_t)threads;
        jb->row_end = nr * (uint64_t)(w + 1) / (uint64_t)threads;
        if (threads == 1) dense_worker(jb);
        else pthread_create(&tid[w], NULL, dense_worker, jb);
    }
    if (threads > 1)
        for (int w = 0; w < threads; ++w) pthread_join(tid[w], NULL);
    free(lhs_rm);
    free(rhs_cm);
    offsets_free(&off);
    return ORC_OK;
}

int orc_mm_dense(const orc_problem *p, int op, int threads) {
    return dense_impl(p, op, 0, p->rows, 0, p->cols, NULL, threads);
}

int orc_mm_dense_block(const orc_problem *p, int op, uint64_t r0, uint64_t nr, uint64_t c0,
                       uint64_t nc, uint32_t *dst, int threads) {
    if (!dst) return ORC_INVALID_ARGUMENT;
    return dense_impl(p, op, r0, nr, c0, nc, dst, threads);
}

/* ------------------------------------------------------------------ Freivalds */
typedef struct {
    const uint32_t *cells;
    const offsets *off;
    uint64_t i0, j0, ncols;
    const uint32_t *vec; /* length ncols */
    uint32_t *res;       /* length rows (slice) */
    uint64_t row_begin, row_end;
    uint32_t q;
} mv_job;

static void *mv_worker(void *arg) {
    mv_job *j = (mv_job *)arg;
    for (uint64_t a = j->row_begin; a < j->row_end; ++a) {
        const uint64_t base = j->off->rowpart[j->i0 + a];
        uint64_t lo = 0, hi = 0;
        uint32_t acc = 0;
        for (uint64_t b = 0; b < j->ncols; ++b) {
            const uint64_t m = j->cells[base + j->off->colpart[j->j0 + b]];
            lo += m * (j->vec[b] & 0xFFFFu);
            hi += m * (j->vec[b] >> 16);
            if ((b & 0xFFFF) == 0xFFFF) {
                acc = (uint32_t)((acc + lo % j->q + (hi % j->q) * ((1ULL << 16) % j->q)) % j->q);
                lo = hi = 0;
            }
        }
        acc = (uint32_t)((acc + lo % j->q + (hi % j->q) * ((1ULL << 16) % j->q)) % j->q);
        j->res[a] = acc;
    }
    return NULL;
}

/* res[a] = sum_b M[i0+a][j0+b] * vec[b] mod q over an nrows x ncols view */
static void matvec(const uint32_t *cells, const offsets *off, uint64_t i0, uint64_t j0,
                   uint64_t nrows, uint64_t ncols, const uint32_t *vec, uint32_t *res,
                   uint32_t q, int threads) {
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > nrows) threads = nrows ? (int)nrows : 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    mv_job jobs[256];
    for (int w = 0; w < threads; ++w) {
        mv_job *jb = &jobs[w];
        jb->cells = cells; jb->off = off; jb->i0 = i0; jb->j0 = j0; jb->ncols = ncols;
        jb->vec = vec; jb->res = res; jb->q = q;
        jb->row_begin = nrows * (uint64_t)w / (uint64_t)threads;
        jb->row_end = nrows * (uint64_t)(w + 1) / (uint64_t)threads;
        if (threads == 1) mv_worker(jb);
        else pthread_create(&tid[w], NULL, mv_worker, jb);
    }
    if (threads > 1)
        for (int w = 0; w < threads; ++w) pthread_join(tid[w], NULL);
}

int orc_freivalds(const orc_problem *p, const uint32_t *new_out, int op, int rounds,
                  uint64_t seed, int threads) {
    int st = check_problem(p);
    if (st) return -st;
    if (op < 0 || op > 2) return -ORC_INVALID_ARGUMENT;
    if (p->rows == 0 || p->cols == 0) return 1;
    const uint64_t n = p->n, t = p->t, q = p->q;
    offsets off;
    if (offsets_make(&off, n, t)) return -100;
    const uint64_t oi = orc_extract_i(n, t, p->out_origin), oj = orc_extract_j(n, t, p->out_origin);
    const uint64_t li = orc_extract_i(n, t, p->lhs_origin), lj = orc_extract_j(n, t, p->lhs_origin);
    const uint64_t ri = orc_extract_i(n, t, p->rhs_origin), rj = orc_extract_j(n, t, p->rhs_origin);
    uint32_t *v = (uint32_t *)malloc(p->cols * sizeof(uint32_t));
    uint32_t *y = (uint32_t *)malloc((p->inner ? p->inner : 1) * sizeof(uint32_t));
    uint32_t *z = (uint32_t *)malloc(p->rows * sizeof(uint32_t));
    uint32_t *w_old = (uint32_t *)malloc(p->rows * sizeof(uint32_t));
    uint32_t *w_new = (uint32_t *)malloc(p->rows * sizeof(uint32_t));
    int ok = 1;
    if (!v || !y || !z || !w_old || !w_new) ok = -100;
    orc_rng g;
    orc_rng_seed(&g, seed);
    for (int rd = 0; rd < rounds && ok == 1; ++rd) {
        for (uint64_t b = 0; b < p->cols; ++b) v[b] = (uint32_t)orc_rng_below(&g, q);
        if (p->inner) {
            matvec(p->rhs, &off, ri, rj, p->inner, p->cols, v, y, (uint32_t)q, threads);
            matvec(p->lhs, &off, li, lj, p->rows, p->inner, y, z, (uint32_t)q, threads);
        } else {
            memset(z, 0, p->rows * sizeof(uint32_t));
        }
        matvec(p->out, &off, oi, oj, p->rows, p->cols, v, w_old, (uint32_t)q, threads);
        matvec(new_out, &off, oi, oj, p->rows, p->cols, v, w_new, (uint32_t)q, threads);
        for (uint64_t a = 0; a < p->rows; ++a) {
            uint64_t want;
            if (op == 0) want = (w_old[a] + (uint64_t)z[a]) % q;
            else if (op == 1) want = (w_old[a] + q - z[a]) % q;
            else want = z[a];
            if (want != w_new[a]) { ok = 0; break; }
        }
    }
    free(v); free(y); free(z); free(w_old); free(w_new);
    offsets_free(&off);
    return ok;
}

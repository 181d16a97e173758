// dropin_test.cpp -- the reference's unit-test scenarios (proj/tests/unit/*.cpp)
// written against the C++ mirror (include/mh/*.hpp) backed by libmhg.so.
// Needs a B200.  Built by __graft_entry__.build(); run by tests/test_cpp_dropin.py.
#include <mh/mh.hpp>

#include <cstdio>
#include <functional>
#include <memory>
#include <algorithm>
#include <random>
#include <set>
#include <string>
#include <vector>

namespace {

int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                               \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(cond)) {                                                            \
            ++g_fail;                                                             \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
        }                                                                         \
    } while (0)

template <typename E, typename F>
bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// test-side dense oracle (oracles.hpp:46-58 semantics)
void dense_acc(mh::Grid& out, const mh::Grid& l, const mh::Grid& r, std::uint64_t oi,
               std::uint64_t oj, std::uint64_t li, std::uint64_t lj, std::uint64_t ri,
               std::uint64_t rj, std::uint64_t rows, std::uint64_t cols, std::uint64_t inner,
               std::uint64_t q, bool sub = false) {
    for (std::uint64_t x = 0; x < rows; ++x)
        for (std::uint64_t y = 0; y < cols; ++y) {
            std::uint64_t acc = out[oi + x][oj + y].v;
            for (std::uint64_t z = 0; z < inner; ++z) {
                std::uint64_t prod = (std::uint64_t(l[li + x][lj + z].v) * r[ri + z][rj + y].v) % q;
                acc = (acc + (sub ? (q - prod) % q : prod)) % q;
            }
            out[oi + x][oj + y] = mh::Fp{std::uint32_t(acc)};
        }
}

mh::Grid random_grid(std::uint64_t n, std::uint32_t q, std::mt19937_64& eng) {
    mh::Grid g(n, std::vector<mh::Fp>(n));
    for (auto& row : g)
        for (auto& cell : row) cell = mh::Fp{std::uint32_t(eng() % q)};
    return g;
}

std::uint64_t shared_segments(std::uint64_t o1, std::uint64_t o2, std::uint64_t len, std::uint64_t t) {
    std::uint64_t c = len ? 1 : 0;
    for (std::uint64_t x = 1; x < len; ++x)
        if ((o1 + x) % t == 0 || (o2 + x) % t == 0) ++c;
    return c;
}

std::uint64_t default_leaves(std::uint64_t d, std::uint64_t t) {
    return d <= t ? 1 : default_leaves((d + 1) / 2, t) + default_leaves(d / 2, t);
}

void test_layout() {
    CHECK(throws_as<std::invalid_argument>([] { mh::Layout(8, 3); }));
    CHECK(throws_as<std::invalid_argument>([] { mh::Layout(12, 4); }));
    CHECK(throws_as<std::invalid_argument>([] { mh::Layout(0, 1); }));
    const mh::Layout p(8, 4);
    CHECK(mh::encode(p, 2, 5) == 25);
    CHECK(mh::encode(p, 5, 6) == 54);
    CHECK(mh::extract_i(p, 47) == 7 && mh::extract_j(p, 47) == 3);
    CHECK(throws_as<std::out_of_range>([&] { mh::encode(p, 8, 0); }));
    CHECK(throws_as<std::invalid_argument>([] { mh::Modulus(9); }));
    const mh::Modulus big(2147483647u);
    CHECK(mh::mul(mh::Fp{2147483646u}, mh::Fp{2147483645u}, big) == mh::Fp{2});
}

void test_split_sub_worked_example() {  // submatrix_test.cpp:100-134
    mh::Matrix m(mh::Layout(8, 4), mh::Modulus(2));
    const mh::Sub s{&m, mh::encode(m.layout(), 1, 2), 4, 4};
    CHECK(s.origin == 6);
    const auto sp = mh::split_sub(mh::Aligned{&m, 0, 64}, s);
    CHECK(sp.rows_north == 3 && sp.cols_west == 2 && sp.rows_south == 1 && sp.cols_east == 2);
    CHECK(sp.part[mh::NW] && sp.part[mh::NW]->origin == 6);
    CHECK(sp.part[mh::NE] && sp.part[mh::NE]->origin == 20);
    CHECK(sp.part[mh::SW] && sp.part[mh::SW]->origin == 34);
    CHECK(sp.part[mh::SE] && sp.part[mh::SE]->origin == 48 && sp.part[mh::SE]->rows == 1);
    CHECK(throws_as<std::logic_error>([&] { mh::quadrants(mh::Aligned{&m, 0, 16}); }));
    CHECK(throws_as<std::out_of_range>([&] { mh::quadrants(mh::Aligned{&m, 16, 64}); }));
    CHECK(throws_as<std::invalid_argument>([&] { mh::quadrants(mh::Aligned{&m, 0, 32}); }));
}

void test_frozen_grid() {  // multiply_test.cpp:134-163
    std::mt19937_64 eng(0);
    const mh::Modulus two(2);
    const mh::Grid ga = random_grid(8, 2, eng), gb = random_grid(8, 2, eng), gc = random_grid(8, 2, eng);
    mh::Matrix A = mh::from_row_major(ga, 4, two), B = mh::from_row_major(gb, 4, two),
               C = mh::from_row_major(gc, 4, two);
    const mh::Layout& p = A.layout();
    mh::mm_naive({mh::Sub{&A, mh::encode(p, 1, 2), 4, 4}, mh::Sub{&B, mh::encode(p, 3, 1), 4, 4},
                  mh::Sub{&C, mh::encode(p, 2, 4), 4, 4}});
    const std::uint32_t frozen[4][4] = {{1, 0, 0, 0}, {1, 0, 1, 1}, {0, 1, 0, 1}, {1, 0, 1, 0}};
    for (int x = 0; x < 4; ++x)
        for (int y = 0; y < 4; ++y) CHECK(A.at(1 + x, 2 + y).v == frozen[x][y]);
    mh::Grid want = ga;
    dense_acc(want, gb, gc, 1, 2, 3, 1, 2, 4, 4, 4, 4, 2);
    CHECK(mh::to_row_major(A) == want);
}

void test_validation() {  // multiply_test.cpp:165-194
    const mh::Modulus two(2);
    mh::Matrix A(mh::Layout(8, 4), two), B(mh::Layout(8, 4), two), C(mh::Layout(8, 4), two);
    CHECK(throws_as<std::logic_error>([&] {
        mh::mm_oblivious({mh::Sub{&A, 0, 4, 4}, mh::Sub{&B, 0, 4, 3}, mh::Sub{&C, 0, 4, 4}});
    }));
    CHECK(throws_as<std::logic_error>([&] {
        mh::mm_oblivious({mh::Sub{&A, 0, 4, 4}, mh::Sub{&A, 0, 4, 4}, mh::Sub{&C, 0, 4, 4}});
    }));
    mh::Matrix D(mh::Layout(8, 4), mh::Modulus(3));
    CHECK(throws_as<std::logic_error>([&] {
        mh::mm_oblivious({mh::Sub{&A, 0, 4, 4}, mh::Sub{&B, 0, 4, 4}, mh::Sub{&D, 0, 4, 4}});
    }));
    mh::Matrix E(mh::Layout(8, 2), two);
    CHECK(throws_as<std::logic_error>([&] {
        mh::mm_oblivious({mh::Sub{&A, 0, 4, 4}, mh::Sub{&B, 0, 4, 4}, mh::Sub{&E, 0, 4, 4}});
    }));
    const mh::Counters c =
        mh::mm_oblivious({mh::Sub{&A, 0, 0, 4}, mh::Sub{&B, 0, 0, 4}, mh::Sub{&C, 0, 4, 4}});
    CHECK(c.base_case_calls == 0 && c.scalar_macs == 0 && c.recursive_calls == 0);
    const mh::Counters one =
        mh::mm_oblivious({mh::Sub{&A, 0, 1, 1}, mh::Sub{&B, 0, 1, 1}, mh::Sub{&C, 0, 1, 1}});
    CHECK(one.base_case_calls == 1 && one.scalar_macs == 1);
    const mh::Counters full = mh::mm_default({mh::Sub{&A, 0, 8, 8}, mh::Sub{&B, 0, 8, 8},
                                              mh::Sub{&C, 0, 8, 8}});
    CHECK(full.base_case_calls == 8 && full.scalar_macs == 512);
}

void test_oblivious_random() {  // multiply_test.cpp:235-268
    std::mt19937_64 eng(44);
    for (int it = 0; it < 30; ++it) {
        const std::uint64_t n = it % 2 ? 16 : 32, t = it % 3 ? 4 : 8;
        const std::uint32_t q = it % 5 ? 2 : 97;
        const std::uint64_t rows = 1 + eng() % n, inner = 1 + eng() % n, cols = 1 + eng() % n;
        const std::uint64_t ia = eng() % (n - rows + 1), ja = eng() % (n - cols + 1);
        const std::uint64_t ib = eng() % (n - rows + 1), jb = eng() % (n - inner + 1);
        const std::uint64_t ic = eng() % (n - inner + 1), jc = eng() % (n - cols + 1);
        const mh::Grid ga = random_grid(n, q, eng), gb = random_grid(n, q, eng),
                       gc = random_grid(n, q, eng);
        const mh::Modulus mod(q);
        mh::Matrix A = mh::from_row_major(ga, t, mod), B = mh::from_row_major(gb, t, mod),
                   C = mh::from_row_major(gc, t, mod);
        const mh::Layout& p = A.layout();
        const mh::Counters ctr =
            mh::mm_oblivious({mh::Sub{&A, mh::encode(p, ia, ja), rows, cols},
                              mh::Sub{&B, mh::encode(p, ib, jb), rows, inner},
                              mh::Sub{&C, mh::encode(p, ic, jc), inner, cols}});
        mh::Grid want = ga;
        dense_acc(want, gb, gc, ia, ja, ib, jb, ic, jc, rows, cols, inner, q);
        CHECK(mh::to_row_major(A) == want);
        CHECK(ctr.scalar_macs == rows * inner * cols);
        CHECK(ctr.encode_calls == 0);
        CHECK(ctr.max_consecutive_jump <= t);
        CHECK(ctr.base_case_calls == shared_segments(ia, ib, rows, t) *
                                         shared_segments(jb, ic, inner, t) *
                                         shared_segments(ja, jc, cols, t));
        std::uint64_t bound = 1, nodes = 1;
        for (unsigned l = 0; l < p.grid_log2; ++l) bound += (nodes *= 64);
        CHECK(ctr.recursive_calls >= ctr.base_case_calls && ctr.recursive_calls <= bound);
        // the same problem as a TU update: C -= A*B on a fresh copy
        mh::Matrix A2 = mh::from_row_major(ga, t, mod);
        mh::mm_oblivious({mh::Sub{&A2, mh::encode(p, ia, ja), rows, cols},
                          mh::Sub{&B, mh::encode(p, ib, jb), rows, inner},
                          mh::Sub{&C, mh::encode(p, ic, jc), inner, cols}},
                         mh::Op::Sub);
        mh::Grid want2 = ga;
        dense_acc(want2, gb, gc, ia, ja, ib, jb, ic, jc, rows, cols, inner, q, true);
        CHECK(mh::to_row_major(A2) == want2);
    }
}

void test_default_leaf_counts() {  // multiply_test.cpp:196-214
    std::mt19937_64 eng(33);
    for (int it = 0; it < 10; ++it) {
        const std::uint64_t n = it % 2 ? 16 : 32, t = it % 3 ? 4 : 8;
        const mh::Modulus two(2);
        mh::Matrix A(mh::Layout(n, t), two), B(mh::Layout(n, t), two), C(mh::Layout(n, t), two);
        const std::uint64_t r = 1 + eng() % n, k = 1 + eng() % n, c = 1 + eng() % n;
        const mh::Counters ctr =
            mh::mm_default({mh::Sub{&A, 0, r, c}, mh::Sub{&B, 0, r, k}, mh::Sub{&C, 0, k, c}});
        CHECK(ctr.base_case_calls == default_leaves(r, t) * default_leaves(k, t) * default_leaves(c, t));
        CHECK(ctr.scalar_macs == r * k * c);
    }
}

void test_host_edits_and_copies() {
    const mh::Modulus q(97);
    mh::Matrix A(mh::Layout(8, 4), q), B(mh::Layout(8, 4), q), C(mh::Layout(8, 4), q);
    for (std::uint64_t i = 0; i < 8; ++i) B.set(i, i, mh::Fp{1});  // identity
    for (mh::Index z = 0; z < 64; ++z) C[z] = mh::Fp{std::uint32_t(z % 97)};
    mh::Matrix A0 = A;  // deep copy
    mh::mm_oblivious({mh::Sub{&A, 0, 8, 8}, mh::Sub{&B, 0, 8, 8}, mh::Sub{&C, 0, 8, 8}});
    CHECK(A == C);
    CHECK(!(A0 == A));
    A[5] = mh::Fp{0};
    mh::mm_oblivious({mh::Sub{&A, 0, 8, 8}, mh::Sub{&B, 0, 8, 8}, mh::Sub{&C, 0, 8, 8}});
    const mh::Matrix& Ar = A;  // reads through the const overload: no host-newer marking
    const mh::Matrix& Cr = C;
    CHECK(Ar[5].v == Cr[5].v && Ar[6].v == (2 * Cr[6].v) % 97);
    // only the touched flat range travels: two pokes 40 cells apart upload 41 cells, a read
    // through the non-const overload one cell, an untouched matrix nothing
    auto uploaded = [](const mh::Matrix& m) {
        std::uint64_t b = 0;
        CHECK(mhg_matrix_upload_bytes(m.device(), &b) == MHG_OK);
        return b;
    };
    A[10] = mh::Fp{3};
    A[50] = mh::Fp{4};
    const std::uint32_t peek = C[7].v;  // non-const access, nothing written
    mh::mm_oblivious({mh::Sub{&A, 0, 8, 8}, mh::Sub{&B, 0, 8, 8}, mh::Sub{&C, 0, 8, 8}});
    CHECK(uploaded(A) == 41 * 4 && uploaded(C) == 4 && peek == 7);
    CHECK(Ar[10].v == (3 + Cr[10].v) % 97 && Ar[50].v == (4 + Cr[50].v) % 97);
    CHECK(Ar[11].v == (3 * Cr[11].v) % 97);  // cells between the pokes kept their device values
}

// ---- re-hosted from proj/tests/unit/multiply_test.cpp:308-437 -------------------------
void test_compatible_parts() {  // multiply_test.cpp:308-361
    const mh::Modulus two(2);
    mh::Matrix A(mh::Layout(8, 4), two), B(mh::Layout(8, 4), two), C(mh::Layout(8, 4), two);
    const mh::Layout& p = A.layout();
    {  // disjoint row ranges yield nothing
        const mh::Framed pa{mh::Sub{&A, mh::encode(p, 0, 0), 3, 2}, 0, 0};
        const mh::Framed pb{mh::Sub{&B, mh::encode(p, 3, 0), 2, 4}, 3, 0};
        const mh::Framed pc{mh::Sub{&C, mh::encode(p, 0, 0), 4, 2}, 0, 0};
        CHECK(!mh::compatible_parts(pa, pb, pc).has_value());
    }
    {  // identical full frames come back unchanged
        const mh::Framed pa{mh::Sub{&A, mh::encode(p, 1, 1), 3, 2}, 0, 0};
        const mh::Framed pb{mh::Sub{&B, mh::encode(p, 2, 2), 3, 4}, 0, 0};
        const mh::Framed pc{mh::Sub{&C, mh::encode(p, 3, 3), 4, 2}, 0, 0};
        const auto got = mh::compatible_parts(pa, pb, pc);
        CHECK(got.has_value());
        for (int op = 0; got && op < 3; ++op) {
            const mh::Framed& in = op == 0 ? pa : op == 1 ? pb : pc;
            const mh::Framed& out = (*got)[op];
            CHECK(out.view.origin == in.view.origin && out.view.rows == in.view.rows &&
                  out.view.cols == in.view.cols && out.row0 == in.row0 && out.col0 == in.col0);
        }
    }
    {  // partial overlaps trim to the intersection box
        const mh::Framed pa{mh::Sub{&A, mh::encode(p, 0, 0), 3, 2}, 0, 0};
        const mh::Framed pb{mh::Sub{&B, mh::encode(p, 1, 0), 2, 4}, 1, 0};
        const mh::Framed pc{mh::Sub{&C, mh::encode(p, 2, 0), 2, 2}, 2, 0};
        const auto got = mh::compatible_parts(pa, pb, pc);
        CHECK(got.has_value());
        if (got) {
            const auto& [ta, tb, tc] = *got;
            CHECK(ta.row0 == 1 && ta.view.rows == 2 && ta.col0 == 0 && ta.view.cols == 2);
            CHECK(ta.view.origin == mh::encode(p, 1, 0));
            CHECK(tb.row0 == 1 && tb.view.rows == 2 && tb.col0 == 2 && tb.view.cols == 2);
            CHECK(tb.view.origin == mh::encode(p, 1, 2));
            CHECK(tc.row0 == 2 && tc.view.rows == 2 && tc.col0 == 0 && tc.view.cols == 2);
            CHECK(tc.view.origin == mh::encode(p, 2, 0));
        }
    }
}

void test_base_case_mm() {  // multiply_test.cpp:363-407
    std::mt19937_64 eng(66);
    const mh::Modulus two(2);
    const mh::Grid ga = random_grid(8, 2, eng), gb = random_grid(8, 2, eng), gc = random_grid(8, 2, eng);
    {  // scattered operand is rejected
        mh::Matrix A = mh::from_row_major(ga, 4, two), B = mh::from_row_major(gb, 4, two),
                   C = mh::from_row_major(gc, 4, two);
        mh::Counters ctr;
        const mh::Sub bad{&B, mh::encode(B.layout(), 2, 2), 4, 4};
        CHECK(!mh::is_contained(bad));
        CHECK(throws_as<std::logic_error>(
            [&] { mh::base_case_mm(mh::Sub{&A, 0, 4, 4}, bad, mh::Sub{&C, 0, 4, 4}, ctr); }));
        CHECK(throws_as<std::logic_error>(  // shapes do not chain
            [&] { mh::base_case_mm(mh::Sub{&A, 0, 4, 4}, mh::Sub{&B, 0, 4, 3}, mh::Sub{&C, 0, 4, 4}, ctr); }));
    }
    {  // single cell: one MAC, empty jump trace
        mh::Matrix A = mh::from_row_major(ga, 4, two), B = mh::from_row_major(gb, 4, two),
                   C = mh::from_row_major(gc, 4, two);
        mh::Counters ctr;
        mh::base_case_mm(mh::Sub{&A, 0, 1, 1}, mh::Sub{&B, 0, 1, 1}, mh::Sub{&C, 0, 1, 1}, ctr);
        CHECK(ctr.base_case_calls == 1 && ctr.scalar_macs == 1);
        CHECK(ctr.max_consecutive_jump == 0 && ctr.encode_calls == 0);
    }
    {  // full tiles: t^3 MACs, jumps within the tile side
        mh::Matrix A = mh::from_row_major(ga, 4, two), B = mh::from_row_major(gb, 4, two),
                   C = mh::from_row_major(gc, 4, two);
        const mh::Layout& p = A.layout();
        mh::Counters ctr;
        mh::base_case_mm(mh::Sub{&A, mh::encode(p, 4, 4), 4, 4}, mh::Sub{&B, mh::encode(p, 4, 0), 4, 4},
                         mh::Sub{&C, mh::encode(p, 0, 4), 4, 4}, ctr);
        CHECK(ctr.scalar_macs == 64);
        CHECK(ctr.max_consecutive_jump <= 4 && ctr.max_consecutive_jump >= 1);
        CHECK(ctr.encode_calls == 0);
        mh::Grid want = ga;
        dense_acc(want, gb, gc, 4, 4, 4, 0, 0, 4, 4, 4, 4, 2);
        CHECK(mh::to_row_major(A) == want);
    }
    {  // result agrees with the dense oracle
        mh::Matrix A = mh::from_row_major(ga, 4, two), B = mh::from_row_major(gb, 4, two),
                   C = mh::from_row_major(gc, 4, two);
        const mh::Layout& p = A.layout();
        mh::Counters ctr;
        mh::Grid want = ga;
        dense_acc(want, gb, gc, 1, 1, 1, 0, 0, 1, 3, 3, 2, 2);
        mh::base_case_mm(mh::Sub{&A, mh::encode(p, 1, 1), 3, 3}, mh::Sub{&B, mh::encode(p, 1, 0), 3, 2},
                         mh::Sub{&C, mh::encode(p, 0, 1), 2, 3}, ctr);
        CHECK(mh::to_row_major(A) == want);
    }
}

// Reference JumpTracker walks (multiply.hpp:80-90, :104-129, :153-170), restated on the
// test side as the checker of the library's closed forms.
struct Walk {
    std::uint64_t last = 0, best = 0;
    bool armed = false;
    void touch(std::uint64_t a) {
        if (armed && a > last && a - last > best) best = a - last;
        last = a;
        armed = true;
    }
};

std::uint64_t encoded_walk(const mh::Layout& la, const mh::Layout& lb, const mh::Layout& lc,
                           std::uint64_t ia, std::uint64_t ja, std::uint64_t ib, std::uint64_t jb,
                           std::uint64_t ic, std::uint64_t jc, std::uint64_t r, std::uint64_t k,
                           std::uint64_t c) {
    Walk ta, tb, tc;
    for (std::uint64_t x = 0; x < r; ++x)
        for (std::uint64_t y = 0; y < c; ++y) {
            ta.touch(mh::encode(la, ia + x, ja + y));
            for (std::uint64_t z = 0; z < k; ++z) {
                tb.touch(mh::encode(lb, ib + x, jb + z));
                tc.touch(mh::encode(lc, ic + z, jc + y));
            }
        }
    return std::max({ta.best, tb.best, tc.best});
}

void default_walk(const mh::Layout& la, const mh::Layout& lb, const mh::Layout& lc, std::uint64_t ia,
                  std::uint64_t ja, std::uint64_t ib, std::uint64_t jb, std::uint64_t ic, std::uint64_t jc,
                  std::uint64_t r, std::uint64_t k, std::uint64_t c, std::uint64_t t, std::uint64_t& best) {
    if (r <= t && k <= t && c <= t) {
        best = std::max(best, encoded_walk(la, lb, lc, ia, ja, ib, jb, ic, jc, r, k, c));
        return;
    }
    const std::uint64_t r1 = r > t ? (r + 1) / 2 : r, c1 = c > t ? (c + 1) / 2 : c, k1 = k > t ? (k + 1) / 2 : k;
    for (int rh = 0; rh < 2; ++rh)
        for (int ch = 0; ch < 2; ++ch)
            for (int kh = 0; kh < 2; ++kh) {
                const std::uint64_t rr = rh ? r - r1 : r1, cc = ch ? c - c1 : c1, kk = kh ? k - k1 : k1;
                const std::uint64_t ro = rh ? r1 : 0, co = ch ? c1 : 0, ko = kh ? k1 : 0;
                if (rr && cc && kk)
                    default_walk(la, lb, lc, ia + ro, ja + co, ib + ro, jb + ko, ic + ko, jc + co, rr, kk, cc, t,
                                 best);
            }
}

void test_naive_default_jumps() {  // multiply.hpp:80-129, 202-230 (mixed layouts allowed)
    std::mt19937_64 eng(99);
    const mh::Modulus q(97);
    for (int it = 0; it < 24; ++it) {
        const std::uint64_t ts[3] = {std::uint64_t(1) << (eng() % 4), std::uint64_t(1) << (eng() % 4),
                                     std::uint64_t(it % 3 ? 4 : 3)};
        std::uint64_t ns[3];
        for (int a = 0; a < 3; ++a) ns[a] = ts[a] << (2 + eng() % 2);
        mh::Matrix A(mh::Layout(ns[0], ts[0]), q), B(mh::Layout(ns[1], ts[1]), q), C(mh::Layout(ns[2], ts[2]), q);
        const std::uint64_t r = 1 + eng() % std::min(ns[0], ns[1]), c = 1 + eng() % std::min(ns[0], ns[2]),
                            k = 1 + eng() % std::min(ns[1], ns[2]);
        const std::uint64_t ia = eng() % (ns[0] - r + 1), ja = eng() % (ns[0] - c + 1);
        const std::uint64_t ib = eng() % (ns[1] - r + 1), jb = eng() % (ns[1] - k + 1);
        const std::uint64_t ic = eng() % (ns[2] - k + 1), jc = eng() % (ns[2] - c + 1);
        const mh::Problem prob{mh::Sub{&A, mh::encode(A.layout(), ia, ja), r, c},
                               mh::Sub{&B, mh::encode(B.layout(), ib, jb), r, k},
                               mh::Sub{&C, mh::encode(C.layout(), ic, jc), k, c}};
        const mh::Counters n = mh::mm_naive(prob);
        CHECK(n.max_consecutive_jump ==
              encoded_walk(A.layout(), B.layout(), C.layout(), ia, ja, ib, jb, ic, jc, r, k, c));
        std::uint64_t best = 0;
        default_walk(A.layout(), B.layout(), C.layout(), ia, ja, ib, jb, ic, jc, r, k, c, ts[0], best);
        const mh::Counters d = mh::mm_default(prob);
        CHECK(d.max_consecutive_jump == best);
        CHECK(n.scalar_macs == r * k * c && d.scalar_macs == r * k * c);
    }
}

void test_scattered_default_run() {  // multiply_test.cpp:409-424
    std::mt19937_64 eng(77);
    const std::uint64_t n = 64, t = 8;
    const mh::Modulus two(2);
    mh::Matrix A = mh::from_row_major(random_grid(n, 2, eng), t, two);
    mh::Matrix B = mh::from_row_major(random_grid(n, 2, eng), t, two);
    mh::Matrix C = mh::from_row_major(random_grid(n, 2, eng), t, two);
    const mh::Index s = mh::encode(A.layout(), t / 2, t / 2);
    const mh::Counters ctr = mh::mm_default({mh::Sub{&A, s, 2 * t, 2 * t}, mh::Sub{&B, s, 2 * t, 2 * t},
                                             mh::Sub{&C, s, 2 * t, 2 * t}});
    CHECK(ctr.max_consecutive_jump > t);
    CHECK(ctr.encode_calls > 0);
}

void test_work_is_exact() {  // multiply_test.cpp:426-437
    std::mt19937_64 eng(88);
    const mh::Modulus q(97);
    for (int it = 0; it < 10; ++it) {
        const std::uint64_t n = 16, t = 4;
        const std::uint64_t r = 1 + eng() % n, k = 1 + eng() % n, c = 1 + eng() % n;
        const mh::Grid ga = random_grid(n, 97, eng), gb = random_grid(n, 97, eng), gc = random_grid(n, 97, eng);
        mh::Matrix B = mh::from_row_major(gb, t, q), C = mh::from_row_major(gc, t, q);
        std::uint64_t res[3];
        mh::Grid out[3];
        for (int kind = 0; kind < 3; ++kind) {
            mh::Matrix A = mh::from_row_major(ga, t, q);
            const mh::Problem prob{mh::Sub{&A, 0, r, c}, mh::Sub{&B, 0, r, k}, mh::Sub{&C, 0, k, c}};
            res[kind] = (kind == 0 ? mh::mm_naive(prob) : kind == 1 ? mh::mm_default(prob)
                                                                    : mh::mm_oblivious(prob)).scalar_macs;
            out[kind] = mh::to_row_major(A);
        }
        CHECK(res[0] == r * k * c && res[1] == r * k * c && res[2] == r * k * c);
        CHECK(out[0] == out[1] && out[1] == out[2]);
    }
}

// ---- re-hosted from proj/tests/unit/submatrix_test.cpp:40-91, 136-249 ----------------
mh::Sub sub_at(mh::Matrix& m, std::uint64_t i, std::uint64_t j, std::uint64_t r, std::uint64_t c) {
    return mh::Sub{&m, mh::encode(m.layout(), i, j), r, c};
}

bool contained_by_scan(const mh::Matrix& m, const mh::Sub& s) {
    const mh::Layout& p = m.layout();
    const auto i0 = mh::extract_i(p, s.origin), j0 = mh::extract_j(p, s.origin);
    std::set<std::pair<std::uint64_t, std::uint64_t>> tiles;
    for (std::uint64_t x = 0; x < s.rows; ++x)
        for (std::uint64_t y = 0; y < s.cols; ++y) tiles.emplace((i0 + x) / p.t, (j0 + y) / p.t);
    return tiles.size() <= 1;
}

void test_alignment_and_containment() {  // submatrix_test.cpp:40-69
    mh::Matrix m16(mh::Layout(16, 4), mh::Modulus(2));
    CHECK(mh::is_aligned(sub_at(m16, 0, 0, 8, 4)));
    CHECK(!mh::is_aligned(sub_at(m16, 1, 2, 4, 4)));
    CHECK(!mh::is_aligned(sub_at(m16, 4, 4, 3, 4)));
    CHECK(mh::is_aligned(sub_at(m16, 4, 8, 4, 8)));
    CHECK(!mh::is_aligned(sub_at(m16, 4, 8, 12, 4)));
    CHECK(!mh::is_aligned(sub_at(m16, 0, 0, 0, 4)));
    mh::Matrix m(mh::Layout(8, 4), mh::Modulus(2));
    CHECK(mh::is_contained(sub_at(m, 0, 0, 4, 4)));
    CHECK(mh::is_contained(sub_at(m, 1, 1, 2, 2)));
    CHECK(!mh::is_contained(sub_at(m, 2, 2, 4, 4)));
    bool all = true;
    for (std::uint64_t i = 0; i < 8; ++i)
        for (std::uint64_t j = 0; j < 8; ++j)
            for (std::uint64_t r = 0; i + r <= 8; ++r)
                for (std::uint64_t c = 0; j + c <= 8; ++c) {
                    const mh::Sub s = sub_at(m, i, j, r, c);
                    all = all && mh::is_contained(s) == contained_by_scan(m, s);
                }
    CHECK(all);
    CHECK(throws_as<std::out_of_range>([&] { mh::is_contained(sub_at(m, 6, 0, 4, 4)); }));
    CHECK(throws_as<std::out_of_range>([&] { mh::is_aligned(mh::Sub{&m, 64, 1, 1}); }));
}

void test_quadrant_order() {  // submatrix_test.cpp:71-91
    mh::Matrix m8(mh::Layout(8, 4), mh::Modulus(2));
    const auto q8 = mh::quadrants(mh::Aligned{&m8, 0, 64});
    for (int t = 0; t < 4; ++t) CHECK(q8[t].origin == std::uint64_t(t) * 16 && q8[t].elems == 16);
    mh::Matrix m16(mh::Layout(16, 4), mh::Modulus(2));
    const auto sh = mh::quadrants(mh::Aligned{&m16, 64, 64});
    CHECK(sh[0].origin == 64 && sh[1].origin == 80 && sh[2].origin == 96 && sh[3].origin == 112);
    const auto top = mh::quadrants(mh::Aligned{&m16, 0, 256});
    CHECK(top[1].origin == 64 && top[2].origin == 128 && top[3].origin == 192 && top[0].elems == 64);
}

void test_split_edge_cases() {  // submatrix_test.cpp:136-168
    mh::Matrix m(mh::Layout(8, 4), mh::Modulus(2));
    const auto sp = mh::split_sub(mh::Aligned{&m, 0, 64}, sub_at(m, 0, 0, 2, 2));
    CHECK(sp.rows_north == 2 && sp.cols_west == 2 && sp.rows_south == 0 && sp.cols_east == 0);
    CHECK(sp.part[mh::NW] && !sp.part[mh::NE] && !sp.part[mh::SW] && !sp.part[mh::SE]);
    const mh::Aligned whole{&m, 0, 64};
    const auto all = mh::split_sub(whole, sub_at(m, 0, 0, 8, 8));
    const auto qs = mh::quadrants(whole);
    for (int t = 0; t < 4; ++t)
        CHECK(all.part[t] && all.part[t]->origin == qs[t].origin && all.part[t]->rows == 4 &&
              all.part[t]->cols == 4);
    mh::Matrix m16(mh::Layout(16, 4), mh::Modulus(2)), other(mh::Layout(16, 4), mh::Modulus(2));
    CHECK(throws_as<std::logic_error>([&] { mh::split_sub(mh::Aligned{&m16, 0, 64}, sub_at(m16, 6, 6, 4, 4)); }));
    CHECK(throws_as<std::invalid_argument>(
        [&] { mh::split_sub(mh::Aligned{&other, 0, 64}, sub_at(m16, 0, 0, 2, 2)); }));
}

// Every view inside every aligned block: split_sub's parts tile it exactly (no gaps,
// no overlap, nothing outside).  submatrix_test.cpp:170-214 / acceptance criterion 2.
bool partition_ok(mh::Matrix& m, const mh::Aligned& a, const mh::Sub& s, std::vector<std::uint32_t>& mark,
                  std::uint32_t& stamp) {
    const mh::Layout& p = m.layout();
    const auto si = mh::extract_i(p, s.origin), sj = mh::extract_j(p, s.origin);
    const auto sp = mh::split_sub(a, s);
    if (sp.rows_north + sp.rows_south != s.rows || sp.cols_west + sp.cols_east != s.cols) return false;
    ++stamp;
    std::uint64_t covered = 0;
    for (const auto& part : sp.part) {
        if (!part) continue;
        const auto pi = mh::extract_i(p, part->origin), pj = mh::extract_j(p, part->origin);
        for (std::uint64_t x = 0; x < part->rows; ++x)
            for (std::uint64_t y = 0; y < part->cols; ++y) {
                if (pi + x < si || pi + x >= si + s.rows || pj + y < sj || pj + y >= sj + s.cols) return false;
                auto& cell = mark[(pi + x) * p.n + (pj + y)];
                if (cell == stamp) return false;
                cell = stamp;
                ++covered;
            }
    }
    return covered == s.rows * s.cols;
}

std::vector<std::uint64_t> tile_sides(std::uint64_t n) {
    std::vector<std::uint64_t> out;
    for (std::uint64_t t = n;; t /= 2) {
        out.push_back(t);
        if (t % 2 != 0) break;
    }
    return out;
}

void test_acceptance_codec() {  // acceptance_main.cpp:43-60 (criterion 1)
    bool ok = true;
    for (std::uint64_t n = 1; n <= 256 && ok; ++n)
        for (std::uint64_t t : tile_sides(n)) {
            const mh::Layout p(n, t);
            std::vector<bool> seen(n * n, false);
            for (std::uint64_t i = 0; i < n && ok; ++i)
                for (std::uint64_t j = 0; j < n; ++j) {
                    std::uint64_t z = 0, ii = 0, jj = 0;
                    // raw C ABI: the codec without exception plumbing per cell
                    ok = ok && mhg_encode(n, t, i, j, &z) == MHG_OK && z < n * n && !seen[z];
                    if (!ok) break;
                    seen[z] = true;
                    ok = ok && mhg_extract(n, t, z, &ii, &jj) == MHG_OK && ii == i && jj == j;
                }
        }
    CHECK(ok);
}

void test_acceptance_partition() {  // acceptance_main.cpp:103-162 (criterion 2), submatrix_test.cpp:170-249
    bool ok = true;
    for (std::uint64_t n = 1; n <= 64 && ok; ++n)
        for (std::uint64_t t : tile_sides(n)) {
            mh::Matrix m(mh::Layout(n, t), mh::Modulus(2));
            const mh::Layout& p = m.layout();
            std::vector<std::uint32_t> mark(n * n, 0);
            std::uint32_t stamp = 0;
            std::mt19937_64 sample_eng(n * 1000 + t);
            for (std::uint64_t elems = p.tile; elems <= p.total && ok; elems *= 4)
                for (std::uint64_t origin = 0; origin < p.total && ok; origin += elems) {
                    const mh::Aligned a{&m, origin, elems};
                    std::vector<mh::Aligned> stack{a};  // recursion ends in whole, contained tiles
                    while (!stack.empty() && ok) {
                        const mh::Aligned blk = stack.back();
                        stack.pop_back();
                        if (blk.elems == p.tile) {
                            ok = blk.origin % p.tile == 0 && mh::is_contained(mh::Sub{&m, blk.origin, p.t, p.t});
                            continue;
                        }
                        for (const auto& child : mh::quadrants(blk)) stack.push_back(child);
                    }
                    if (elems == p.tile) {  // views inside a tile-level block are contained
                        const auto bi = mh::extract_i(p, origin), bj = mh::extract_j(p, origin);
                        if (n <= 8)
                            for (std::uint64_t di = 0; di < p.t; ++di)
                                for (std::uint64_t dj = 0; dj < p.t; ++dj)
                                    for (std::uint64_t r = 1; di + r <= p.t; ++r)
                                        for (std::uint64_t c = 1; dj + c <= p.t; ++c)
                                            ok = ok && mh::is_contained(sub_at(m, bi + di, bj + dj, r, c));
                        continue;
                    }
                    const auto side = mh::aligned_side(a);
                    const auto ai = mh::extract_i(p, origin), aj = mh::extract_j(p, origin);
                    if (n <= 16) {
                        for (std::uint64_t si = ai; si < ai + side && ok; ++si)
                            for (std::uint64_t sj = aj; sj < aj + side && ok; ++sj)
                                for (std::uint64_t r = 1; si + r <= ai + side && ok; ++r)
                                    for (std::uint64_t c = 1; sj + c <= aj + side && ok; ++c)
                                        ok = partition_ok(m, a, sub_at(m, si, sj, r, c), mark, stamp);
                    } else {
                        ok = partition_ok(m, a, mh::Sub{&m, origin, side, side}, mark, stamp);
                        for (int k = 0; k < 8 && ok; ++k) {
                            const auto r = 1 + sample_eng() % side, c = 1 + sample_eng() % side;
                            const auto si = ai + sample_eng() % (side - r + 1), sj = aj + sample_eng() % (side - c + 1);
                            ok = partition_ok(m, a, sub_at(m, si, sj, r, c), mark, stamp);
                        }
                    }
                }
        }
    CHECK(ok);
}

// TU/TURBO Schur-update driver (include/mh/tu.hpp): a right-looking
// sweep on ONE parent with a misaligned panel width equals the dense elimination loop,
// through the one-shot aliased update and through the planned sweep (run twice: the
// second run continues from the first one's cells).
void test_tu_schur_sweep() {
    std::mt19937_64 eng(77);
    const std::uint64_t n = 256, t = 32, block = 40;
    const std::uint32_t q = 65521;
    const mh::Modulus mod(q);
    mh::Grid g = random_grid(n, q, eng);
    auto dense_sweep = [&](mh::Grid& d) {
        for (std::uint64_t k0 = 0; k0 + block < n; k0 += block) {
            const std::uint64_t k1 = k0 + block, rest = n - k1;
            const mh::Grid snap = d;  // operands are disjoint from the output: same as in place
            dense_acc(d, snap, snap, k1, k1, k1, k0, k0, k1, rest, rest, block, q, true);
        }
    };
    mh::Grid want = g;
    dense_sweep(want);
    // one-shot aliased updates
    mh::Matrix A = mh::from_row_major(g, t, mod);
    std::uint64_t macs = 0;
    const auto steps = mh::tu::schur_views(A, block);
    CHECK(steps.size() == 6);
    for (const mh::Problem& p : steps) {
        const mh::Counters c = mh::tu::schur_update(p);
        CHECK(c.scalar_macs == p.a.rows * p.a.cols * p.b.cols);
        CHECK(c.encode_calls == 0);
        macs += c.scalar_macs;
    }
    CHECK(mh::to_row_major(A) == want);
    // the reference's entry point still refuses the shared parent
    CHECK(throws_as<std::logic_error>([&] { mh::mm_oblivious(steps[0]); }));
    // planned sweep, replayed
    mh::Matrix B = mh::from_row_major(g, t, mod);
    mh::tu::SchurSweep sweep(B, block);
    CHECK(sweep.steps() == 6 && sweep.macs() == macs);
    CHECK(sweep.run() == macs);
    CHECK(mh::to_row_major(B) == want);
    mh::Grid want2 = want;
    dense_sweep(want2);
    B.set(0, 0, B.at(0, 0));  // a host-side touch between runs is uploaded, not lost
    sweep.run();
    CHECK(mh::to_row_major(B) == want2);
    // add form and argument checks
    mh::Matrix C = mh::from_row_major(g, t, mod);
    mh::Grid want3 = g;
    dense_acc(want3, g, g, 64, 64, 64, 0, 0, 64, 192, 192, 64, q, false);
    mh::tu::schur_update(mh::Problem{mh::Sub{&C, mh::encode(C.layout(), 64, 64), 192, 192},
                                     mh::Sub{&C, mh::encode(C.layout(), 64, 0), 192, 64},
                                     mh::Sub{&C, mh::encode(C.layout(), 0, 64), 64, 192}},
                         mh::Op::Add);
    CHECK(mh::to_row_major(C) == want3);
    CHECK(throws_as<std::invalid_argument>([&] { mh::tu::schur_views(C, 0); }));
    CHECK(mh::tu::schur_views(C, n).empty());
    CHECK(throws_as<std::logic_error>([&] {
        mh::tu::schur_update(mh::Problem{mh::Sub{&C, 0, 8, 8}, mh::Sub{&C, 0, 8, 4}, mh::Sub{&C, 0, 5, 8}});
    }));
}

// Multi-GPU partition through the C ABI (mhg_dist_*), driven the way a C++ host
// program would: every rank's K-segment plans (packs + GEMM run separately, as around a
// broadcast of the packed bytes), here all on one device, make the whole multiply.
void test_dist_segment_plans() {
    std::mt19937_64 eng(404);
    const std::uint64_t n = 256, t = 32;
    const std::uint32_t q = 65521, P = 8;
    const mh::Modulus mod(q);
    const mh::Grid gc = random_grid(n, q, eng), ga = random_grid(n, q, eng), gb = random_grid(n, q, eng);
    mh::Matrix C = mh::from_row_major(gc, t, mod), A = mh::from_row_major(ga, t, mod),
               B = mh::from_row_major(gb, t, mod);
    std::uint32_t nseg = 0;
    CHECK(mhg_dist_segment_count(P, &nseg) == MHG_OK && nseg == 4);
    std::uint64_t cells = 0, macs = 0;
    for (std::uint32_t r = 0; r < P; ++r) {
        mhg_dist_block_t blk{};
        CHECK(mhg_dist_block(P, r, n, t, &blk) == MHG_OK);
        std::uint64_t lo = 0, hi = 0;
        CHECK(mhg_dist_slice(P, r, n, &lo, &hi) == MHG_OK);
        CHECK(hi - lo == blk.rows * blk.cols && lo == mh::encode(C.layout(), blk.i0, blk.j0));
        cells += hi - lo;
        for (std::uint32_t s = 0; s < nseg; ++s) {
            mhg_dist_segment_t sg{};
            CHECK(mhg_dist_segment(P, r, n, t, s, &sg) == MHG_OK);
            CHECK(sg.a_begin == mh::encode(A.layout(), blk.i0, sg.k0));
            CHECK(sg.b_begin == mh::encode(B.layout(), sg.k0, blk.j0));
            mhg_plan pl = nullptr;
            CHECK(mhg_dist_plan_create(C.device(), A.device(), B.device(), MHG_OP_SUB, P, r, s, &pl) == MHG_OK);
            if (!pl) continue;
            mhg_counters c{};
            CHECK(mhg_plan_counters(pl, &c) == MHG_OK);
            macs += c.scalar_macs;
            // the owner's packs, (the broadcast of mhg_plan_pack_buffer goes here), the GEMM
            CHECK(mhg_plan_pack(pl, 0, nullptr) == MHG_OK && mhg_plan_pack(pl, 1, nullptr) == MHG_OK);
            void* ptr = nullptr;
            std::uint64_t bytes = 0;
            CHECK(mhg_plan_pack_buffer(pl, 0, &ptr, &bytes) == MHG_OK && ptr && bytes);
            CHECK(mhg_plan_gemm(pl, nullptr) == MHG_OK);
            CHECK(mhg_synchronize(nullptr) == MHG_OK);
            mhg_plan_destroy(pl);
        }
    }
    C.device_written();
    CHECK(cells == n * n && macs == n * n * n);
    mh::Grid want = gc;
    dense_acc(want, ga, gb, 0, 0, 0, 0, 0, 0, n, n, n, q, true);
    CHECK(mh::to_row_major(C) == want);
    mhg_dist_block_t blk{};
    CHECK(mhg_dist_block(6, 0, n, t, &blk) == MHG_ERR_INVALID_ARGUMENT);
    CHECK(mhg_dist_block(4, 4, n, t, &blk) == MHG_ERR_OUT_OF_RANGE);
}

// The explicit-stream variant (SURVEY 8(b) threading): the call returns after enqueueing,
// host-side reads of the output wait for it, host edits made after it are uploaded before
// the next multiply, and a chain of asynchronous calls equals the synchronous results.
void test_async_variant() {
    std::mt19937_64 eng(909);
    const std::uint64_t n = 256, t = 32;
    const std::uint32_t q = 65521;
    const mh::Modulus mod(q);
    mh::Grid gc = random_grid(n, q, eng);
    const mh::Grid ga = random_grid(n, q, eng), gb = random_grid(n, q, eng);
    mh::Matrix C = mh::from_row_major(gc, t, mod), A = mh::from_row_major(ga, t, mod),
               B = mh::from_row_major(gb, t, mod);
    const mh::Problem p{mh::Sub{&C, mh::encode(C.layout(), 17, 40), 200, 150},
                        mh::Sub{&A, mh::encode(A.layout(), 3, 9), 200, 120},
                        mh::Sub{&B, mh::encode(B.layout(), 77, 5), 120, 150}};
    const mh::Counters c1 = mh::mm_oblivious_async(p, mh::Op::Sub);
    const mh::Counters c2 = mh::mm_oblivious_async(p);  // Add, same stream: ordered after the first
    CHECK(c1.scalar_macs == 200ull * 150 * 120 && c2.base_case_calls == c1.base_case_calls);
    CHECK(mh::to_row_major(C) == gc);  // -AB then +AB: back to the start; the read waited
    // a host edit after the asynchronous calls reaches the device before the next one
    C.set(17, 40, mh::Fp{5});
    gc[17][40] = mh::Fp{5};
    mh::mm_oblivious_async(p, mh::Op::Sub);
    mh::synchronize();
    dense_acc(gc, ga, gb, 17, 40, 3, 9, 77, 5, 200, 150, 120, q, true);
    CHECK(mh::to_row_major(C) == gc);
    // same validation as the synchronous entry point
    CHECK(throws_as<std::logic_error>([&] {
        mh::mm_oblivious_async(mh::Problem{p.a, mh::Sub{&C, 0, 200, 120}, p.c});
    }));
    // the reference's concurrency contract (multiply.hpp:25-29): two multiplies on disjoint
    // output rectangles of one container, in flight on two non-blocking streams
    void *s1 = nullptr, *s2 = nullptr;
    CHECK(mhg_stream_create(&s1, 1) == MHG_OK && mhg_stream_create(&s2, 1) == MHG_OK && s1 && s2);
    mh::Matrix A2 = mh::from_row_major(ga, t, mod), B2 = mh::from_row_major(gb, t, mod);
    mh::Grid want = mh::to_row_major(C);
    const mh::Problem top{mh::Sub{&C, mh::encode(C.layout(), 0, 0), 100, 256},
                          mh::Sub{&A, mh::encode(A.layout(), 5, 0), 100, 256},
                          mh::Sub{&B, mh::encode(B.layout(), 0, 0), 256, 256}};
    const mh::Problem bottom{mh::Sub{&C, mh::encode(C.layout(), 100, 0), 156, 256},
                             mh::Sub{&A2, mh::encode(A2.layout(), 50, 0), 156, 256},
                             mh::Sub{&B2, mh::encode(B2.layout(), 0, 0), 256, 256}};
    for (int rep = 0; rep < 3; ++rep) {
        mh::mm_oblivious_async(top, mh::Op::Add, s1);
        mh::mm_oblivious_async(bottom, mh::Op::Sub, s2);  // both write C (disjoint rows): concurrent
        dense_acc(want, ga, gb, 0, 0, 5, 0, 0, 0, 100, 256, 256, q, false);
        dense_acc(want, ga, gb, 100, 0, 50, 0, 0, 0, 156, 256, 256, q, true);
    }
    CHECK(mh::to_row_major(C) == want);  // the read waits for both streams C is in flight on
    // a dependent call on another stream: B2 = B2 + C * A2-like chain -- reading C on s2 waits
    // for its writers on s1
    mh::Matrix D = mh::from_row_major(gc, t, mod);
    const mh::Problem into_c{mh::Sub{&C, 0, 64, 64}, mh::Sub{&A, 0, 64, 64}, mh::Sub{&B, 0, 64, 64}};
    const mh::Problem from_c{mh::Sub{&D, 0, 64, 64}, mh::Sub{&C, 0, 64, 64}, mh::Sub{&B2, 0, 64, 64}};
    mh::mm_oblivious_async(into_c, mh::Op::Add, s1);
    mh::mm_oblivious_async(from_c, mh::Op::Add, s2);
    dense_acc(want, ga, gb, 0, 0, 0, 0, 0, 0, 64, 64, 64, q, false);
    mh::Grid want_d = gc;
    dense_acc(want_d, want, gb, 0, 0, 0, 0, 0, 0, 64, 64, 64, q, false);
    CHECK(mh::to_row_major(D) == want_d && mh::to_row_major(C) == want);
    mh::synchronize(s1);
    mh::synchronize(s2);
    CHECK(mhg_stream_destroy(s1) == MHG_OK && mhg_stream_destroy(s2) == MHG_OK);
}

// detail::dilate / undilate (layout.hpp:15-33) against the codec, and detail::JumpTracker
// (multiply.hpp:80-90) measuring base_case_mm's walk against its closed-form counter.
void test_detail_helpers() {
    const mh::Layout lay(64, 4);
    for (std::uint64_t i = 0; i < 64; i += 3)
        for (std::uint64_t j = 0; j < 64; j += 5) {
            const std::uint64_t z = ((mh::detail::dilate(lay.tdiv(i)) << 1) | mh::detail::dilate(lay.tdiv(j))) * lay.tile +
                                    lay.tmod(i) * lay.t + lay.tmod(j);
            CHECK(z == mh::encode(lay, i, j));
            CHECK(mh::detail::undilate(lay.tilediv(z) >> 1) == lay.tdiv(i));
            CHECK(mh::detail::undilate(lay.tilediv(z)) == lay.tdiv(j));
        }
    // the walk of a contained leaf (out 3 x 2, inner 4, t = 8), tracked cell by cell
    const mh::Modulus mod(97);
    mh::Matrix A(mh::Layout(16, 8), mod), B(mh::Layout(16, 8), mod), C(mh::Layout(16, 8), mod);
    const mh::Sub out{&A, mh::encode(A.layout(), 1, 2), 3, 2}, lhs{&B, mh::encode(B.layout(), 9, 1), 3, 4},
        rhs{&C, mh::encode(C.layout(), 2, 10), 4, 2};
    mh::Counters walked{}, closed{};
    mh::detail::JumpTracker ja, jb, jc;
    for (std::uint64_t x = 0; x < 3; ++x)
        for (std::uint64_t y = 0; y < 2; ++y) {
            ja.touch(out.origin + x * 8 + y, walked);
            for (std::uint64_t z = 0; z < 4; ++z) {
                jb.touch(lhs.origin + x * 8 + z, walked);
                jc.touch(rhs.origin + z * 8 + y, walked);
            }
        }
    mh::base_case_mm(out, lhs, rhs, closed);
    CHECK(walked.max_consecutive_jump == closed.max_consecutive_jump);
    CHECK(closed.max_consecutive_jump == 8);
}

}  // namespace

int main() {
    const std::pair<const char*, std::function<void()>> tests[] = {
        {"layout", test_layout},
        {"split_sub", test_split_sub_worked_example},
        {"frozen_grid", test_frozen_grid},
        {"validation", test_validation},
        {"oblivious_random", test_oblivious_random},
        {"default_leaf_counts", test_default_leaf_counts},
        {"host_edits_and_copies", test_host_edits_and_copies},
        {"compatible_parts", test_compatible_parts},
        {"base_case_mm", test_base_case_mm},
        {"naive_default_jumps", test_naive_default_jumps},
        {"scattered_default_run", test_scattered_default_run},
        {"work_is_exact", test_work_is_exact},
        {"alignment_and_containment", test_alignment_and_containment},
        {"quadrant_order", test_quadrant_order},
        {"split_edge_cases", test_split_edge_cases},
        {"acceptance_codec", test_acceptance_codec},
        {"acceptance_partition", test_acceptance_partition},
        {"tu_schur_sweep", test_tu_schur_sweep},
        {"dist_segment_plans", test_dist_segment_plans},
        {"async_variant", test_async_variant},
        {"detail_helpers", test_detail_helpers},
    };
    for (const auto& [name, fn] : tests) {
        const int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::fprintf(stderr, "FAIL %s: exception %s\n", name, e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
        std::fflush(stdout);  // keep the log if a later test dies
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}

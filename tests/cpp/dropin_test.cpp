// dropin_test.cpp -- the reference's unit-test scenarios (proj/tests/unit/*.cpp)
// written against the C++ mirror (include/mh/*.hpp) backed by libmhg.so.
// Needs a B200.  Built by __graft_entry__.build(); run by tests/test_cpp_dropin.py.
#include <mh/mh.hpp>

#include <cstdio>
#include <functional>
#include <memory>
#include <random>
#include <string>

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
    CHECK(A[5].v == C[5].v && A[6].v == (2 * C[6].v) % 97);
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
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}

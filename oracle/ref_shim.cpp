// ref_shim.cpp -- C ABI over the UNMODIFIED reference library (header-only,
// compiled in place from /root/reference/proj/include with the reference's
// Release flags -std=c++20 -O3 -DNDEBUG; see oracle/Makefile).
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Output goes to oracle/_ref/libmhref.so
// (git-ignored).  It serves two roles:
//   1. pins the C restatement (oracle/mh_oracle.c) and the golden fixtures
//      against the reference itself;
//   2. the reference CPU arm of bench.py (--impl reference / cpu_baseline):
//      mh::mm_oblivious run over disjoint output strips on std::threads, as
//      the reference's concurrency contract allows (multiply.hpp:25-29).
#include <mh/mh.hpp>

#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

namespace {

struct Counters5 {
    std::uint64_t base_case_calls, scalar_macs, encode_calls, recursive_calls, max_consecutive_jump;
};

void put(const mh::Counters& c, Counters5* out) {
    if (!out) return;
    out->base_case_calls = c.base_case_calls;
    out->scalar_macs = c.scalar_macs;
    out->encode_calls = c.encode_calls;
    out->recursive_calls = c.recursive_calls;
    out->max_consecutive_jump = c.max_consecutive_jump;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (const std::logic_error&) {
        return 3;
    } catch (...) {
        return 4;
    }
}

void load(mh::Matrix& m, const std::uint32_t* cells) {
    auto& v = m.cells();
    for (std::size_t z = 0; z < v.size(); ++z) v[z] = mh::Fp{cells[z]};
}

void store(const mh::Matrix& m, std::uint32_t* cells) {
    const auto& v = m.cells();
    for (std::size_t z = 0; z < v.size(); ++z) cells[z] = v[z].v;
}

}  // namespace

extern "C" {

int ref_encode(std::uint64_t n, std::uint64_t t, std::uint64_t i, std::uint64_t j,
               std::uint64_t* z) {
    return guarded([&] { *z = mh::encode(mh::Layout(n, t), i, j); });
}

int ref_extract(std::uint64_t n, std::uint64_t t, std::uint64_t z, std::uint64_t* i,
                std::uint64_t* j) {
    return guarded([&] {
        const mh::Layout lay(n, t);
        *i = mh::extract_i(lay, z);
        *j = mh::extract_j(lay, z);
    });
}

// kind: 0 mm_naive, 1 mm_default, 2 mm_oblivious.
// op:   0 out += lhs*rhs (the reference semantics),
//       1 out -= lhs*rhs computed as out += (-lhs)*rhs on a negated copy,
//       2 out  = lhs*rhs computed by zeroing the view cells, then +=.
int ref_mm(int kind, std::uint64_t n, std::uint64_t t, std::uint32_t q, std::uint32_t* out,
           std::uint64_t out_origin, std::uint64_t rows, std::uint64_t cols,
           const std::uint32_t* lhs, std::uint64_t lhs_origin, std::uint64_t inner,
           const std::uint32_t* rhs, std::uint64_t rhs_origin, int op, Counters5* ctr) {
    return guarded([&] {
        const mh::Layout lay(n, t);
        const mh::Modulus mod(q);
        mh::Matrix A(lay, mod), B(lay, mod), C(lay, mod);
        load(A, out);
        load(B, lhs);
        load(C, rhs);
        if (op == 1)
            for (auto& v : B.cells()) v.v = v.v ? q - v.v : 0;
        const mh::Problem prob{mh::Sub{&A, out_origin, rows, cols},
                               mh::Sub{&B, lhs_origin, rows, inner},
                               mh::Sub{&C, rhs_origin, inner, cols}};
        if (op == 2) {
            mh::check_sub(prob.a);
            const std::uint64_t i0 = mh::extract_i(lay, out_origin), j0 = mh::extract_j(lay, out_origin);
            for (std::uint64_t x = 0; x < rows; ++x)
                for (std::uint64_t y = 0; y < cols; ++y) A.set(i0 + x, j0 + y, mh::Fp{0});
        }
        mh::Counters c;
        if (kind == 0) c = mh::mm_naive(prob);
        else if (kind == 1) c = mh::mm_default(prob);
        else c = mh::mm_oblivious(prob);
        put(c, ctr);
        store(A, out);
    });
}

// Counters of mm_naive (kind 0) / mm_default (kind 1) on three containers that may
// differ in layout (the reference allows it for these two): zero-filled GF(2) stores,
// only the Counters are reported.
int ref_counters_mixed(int kind, std::uint64_t na, std::uint64_t ta, std::uint64_t oa,
                       std::uint64_t nb, std::uint64_t tb, std::uint64_t ob, std::uint64_t nc,
                       std::uint64_t tc, std::uint64_t oc, std::uint64_t rows, std::uint64_t inner,
                       std::uint64_t cols, Counters5* ctr) {
    return guarded([&] {
        const mh::Modulus two(2);
        mh::Matrix A(mh::Layout(na, ta), two), B(mh::Layout(nb, tb), two), C(mh::Layout(nc, tc), two);
        const mh::Problem prob{mh::Sub{&A, oa, rows, cols}, mh::Sub{&B, ob, rows, inner},
                               mh::Sub{&C, oc, inner, cols}};
        put(kind == 0 ? mh::mm_naive(prob) : mh::mm_default(prob), ctr);
    });
}

// The reference's text writer (io.hpp:16-26, save_matrix_file :52-57) on a container
// filled from mh::Rng(seed) in flat Morton order.
int ref_save_matrix(std::uint64_t n, std::uint64_t t, std::uint32_t q, std::uint64_t seed, const char* path) {
    return guarded([&] {
        mh::Matrix m(mh::Layout(n, t), mh::Modulus(q));
        mh::Rng rng(seed);
        for (auto& v : m.cells()) v = mh::Fp{std::uint32_t(rng.below(q))};
        mh::save_matrix_file(path, m);
    });
}

// Draw the (skip+1)-th instance of Rng(seed) exactly as gen_problem does.
int ref_gen_problem(std::uint64_t n, std::uint64_t t, std::uint32_t q, std::uint64_t seed,
                    std::uint32_t skip, std::uint32_t* out, std::uint32_t* lhs,
                    std::uint32_t* rhs, std::uint64_t desc[10]) {
    return guarded([&] {
        mh::Config cfg;
        cfg.n = n;
        cfg.t = t;
        cfg.q = q;
        cfg.seed = seed;
        mh::Rng rng(seed);
        for (std::uint32_t s = 0; s < skip; ++s) (void)mh::gen_problem(cfg, rng);
        const mh::Instance inst = mh::gen_problem(cfg, rng);
        store(*inst.a, out);
        store(*inst.b, lhs);
        store(*inst.c, rhs);
        desc[0] = inst.aligned_draw;
        desc[1] = inst.sa.origin; desc[2] = inst.sa.rows; desc[3] = inst.sa.cols;
        desc[4] = inst.sb.origin; desc[5] = inst.sb.rows; desc[6] = inst.sb.cols;
        desc[7] = inst.sc.origin; desc[8] = inst.sc.rows; desc[9] = inst.sc.cols;
    });
}

// algo: 0 default, 1 oblivious, 2 both (bench.hpp:23)
int ref_run_trials_csv(std::uint64_t n, std::uint64_t t, std::uint32_t q, std::uint64_t seed,
                       std::uint32_t trials, int algo, const char* path) {
    return guarded([&] {
        mh::Config cfg;
        cfg.n = n;
        cfg.t = t;
        cfg.q = q;
        cfg.seed = seed;
        cfg.trials = trials;
        cfg.algo = algo == 0 ? mh::Algo::Default : algo == 1 ? mh::Algo::Oblivious : mh::Algo::Both;
        mh::write_trials_csv(mh::run_trials(cfg), path);
    });
}

// ------------------------------------------------------------- CPU baseline
struct RefBench {
    mh::Layout lay;
    mh::Modulus mod;
    std::unique_ptr<mh::Matrix> out, lhs, rhs;
};

// Three n x n containers filled exactly as the reference's gen_problem fills them
// (bench.hpp:101-103): one mh::Rng(seed) stream, below(q) per cell in flat Morton
// order, out then lhs then rhs -- the same residues bench.py's GPU arm multiplies.
void* ref_bench_new(std::uint64_t n, std::uint64_t t, std::uint32_t q, std::uint64_t seed) {
    try {
        auto* b = new RefBench{mh::Layout(n, t), mh::Modulus(q), nullptr, nullptr, nullptr};
        b->out = std::make_unique<mh::Matrix>(b->lay, b->mod);
        b->lhs = std::make_unique<mh::Matrix>(b->lay, b->mod);
        b->rhs = std::make_unique<mh::Matrix>(b->lay, b->mod);
        mh::Rng rng(seed);
        for (mh::Matrix* m : {b->out.get(), b->lhs.get(), b->rhs.get()})
            for (auto& v : m->cells()) v = mh::Fp{std::uint32_t(rng.below(q))};
        return b;
    } catch (...) {
        return nullptr;
    }
}

void ref_bench_free(void* h) { delete static_cast<RefBench*>(h); }

// Time mm_oblivious on the output block rows [i0, i0+rows) x cols [j0, j0+cols)
// with full inner dimension `inner` starting at lhs column / rhs row k0,
// split into `threads` disjoint row strips (each strip its own mm_oblivious
// call on its own thread).  Returns wall ns, or a negative status.
long long ref_bench_run(void* h, std::uint64_t i0, std::uint64_t rows, std::uint64_t j0,
                        std::uint64_t cols, std::uint64_t k0, std::uint64_t inner, int threads,
                        std::uint64_t* macs) {
    auto* b = static_cast<RefBench*>(h);
    if (!b || threads < 1) return -1;
    const mh::Layout& lay = b->lay;
    std::vector<mh::Problem> parts;
    const std::uint64_t tside = lay.t;
    // strips are cut on tile boundaries when possible (each strip a separate call)
    for (int w = 0; w < threads; ++w) {
        std::uint64_t a = rows * std::uint64_t(w) / std::uint64_t(threads);
        std::uint64_t e = rows * std::uint64_t(w + 1) / std::uint64_t(threads);
        if (rows >= tside * std::uint64_t(threads)) {
            a = a / tside * tside;
            e = (w + 1 == threads) ? rows : e / tside * tside;
        }
        if (e <= a) continue;
        parts.push_back(mh::Problem{mh::Sub{b->out.get(), mh::encode(lay, i0 + a, j0), e - a, cols},
                                    mh::Sub{b->lhs.get(), mh::encode(lay, i0 + a, k0), e - a, inner},
                                    mh::Sub{b->rhs.get(), mh::encode(lay, k0, j0), inner, cols}});
    }
    std::vector<std::uint64_t> work(parts.size(), 0);
    std::vector<std::thread> pool;
    const auto t0 = std::chrono::steady_clock::now();
    for (std::size_t w = 0; w < parts.size(); ++w)
        pool.emplace_back([&, w] { work[w] = mh::mm_oblivious(parts[w]).scalar_macs; });
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (macs) {
        *macs = 0;
        for (auto v : work) *macs += v;
    }
    return std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
}

}  // extern "C"

// mh/multiply.hpp -- the multiply entry points (reference: multiply.hpp:39-308).
//
// mm_oblivious is the drop-in: identical results (the whole output container,
// bit for bit) and identical Counters, computed by libmhg.so's int8 limb-split
// tcgen05 kernels; the Counters come from the planner's closed form of the
// oblivious recursion.  Calls are synchronous like the reference's.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <tuple>

#include "mh/submatrix.hpp"

namespace mh {

struct Counters {
    std::uint64_t base_case_calls = 0;
    std::uint64_t scalar_macs = 0;
    std::uint64_t encode_calls = 0;
    std::uint64_t recursive_calls = 0;
    std::uint64_t max_consecutive_jump = 0;
};

/// a (output) += b (left) * c (right), each view in its own container.
struct Problem {
    Sub a;
    Sub b;
    Sub c;
};

/// Operation on the output view (the reference only has Add).
enum class Op { Add = MHG_OP_ADD, Sub = MHG_OP_SUB, Set = MHG_OP_SET };

inline void check_problem(const Problem& p) {
    check_sub(p.a);
    check_sub(p.b);
    check_sub(p.c);
    if (p.a.mat == p.b.mat || p.a.mat == p.c.mat || p.b.mat == p.c.mat)
        throw std::logic_error("problem: the three views must live in distinct matrices");
    if (p.a.rows != p.b.rows || p.a.cols != p.c.cols || p.b.cols != p.c.rows)
        throw std::logic_error("problem: view shapes do not chain");
    if (p.a.mat->modulus().q != p.b.mat->modulus().q || p.a.mat->modulus().q != p.c.mat->modulus().q)
        throw std::logic_error("problem: operands use different moduli");
}

/// A view plus its rectangle's position on the problem's shared axes.
struct Framed {
    Sub view;
    std::uint64_t row0 = 0;
    std::uint64_t col0 = 0;
};

/// Step 4: trim three framed pieces to their shared row / inner / column ranges.
inline std::optional<std::array<Framed, 3>> compatible_parts(const Framed& pa, const Framed& pb,
                                                             const Framed& pc) {
    struct Range {
        std::uint64_t lo, hi;
    };
    auto meet = [](std::uint64_t a0, std::uint64_t an, std::uint64_t b0, std::uint64_t bn) {
        return Range{std::max(a0, b0), std::min(a0 + an, b0 + bn)};
    };
    const Range x = meet(pa.row0, pa.view.rows, pb.row0, pb.view.rows);
    const Range z = meet(pb.col0, pb.view.cols, pc.row0, pc.view.rows);
    const Range y = meet(pa.col0, pa.view.cols, pc.col0, pc.view.cols);
    if (x.hi <= x.lo || z.hi <= z.lo || y.hi <= y.lo) return std::nullopt;
    auto trim = [](const Framed& f, Range r, Range c) {
        const Layout& lay = f.view.mat->layout();
        const std::uint64_t i = extract_i(lay, f.view.origin) + (r.lo - f.row0);
        const std::uint64_t j = extract_j(lay, f.view.origin) + (c.lo - f.col0);
        return Framed{Sub{f.view.mat, encode(lay, i, j), r.hi - r.lo, c.hi - c.lo}, r.lo, c.lo};
    };
    return std::array<Framed, 3>{trim(pa, x, y), trim(pb, x, z), trim(pc, z, y)};
}

namespace gpu {

inline mhg_view view_of(const Sub& s) { return mhg_view{s.mat->device(), s.origin, s.rows, s.cols}; }

inline Counters to_counters(const mhg_counters& c) {
    return Counters{c.base_case_calls, c.scalar_macs, c.encode_calls, c.recursive_calls,
                    c.max_consecutive_jump};
}

/// out op= lhs * rhs on the device, synchronous; returns the oblivious Counters.
inline Counters run(const Problem& p, Op op) {
    check_problem(p);
    mhg_counters c{};
    gpu::check(mhg_mm(view_of(p.a), view_of(p.b), view_of(p.c), static_cast<mhg_op>(op), &c,
                      nullptr));
    gpu::check(mhg_synchronize(nullptr));
    p.a.mat->device_written();
    return to_counters(c);
}

}  // namespace gpu

/// Drop-in for the reference's mm_oblivious (multiply.hpp:297-308).
inline Counters mm_oblivious(const Problem& p) { return gpu::run(p, Op::Add); }

/// Same engine with the TU/TURBO operations: Op::Sub is C -= A*B, Op::Set is C = A*B.
inline Counters mm_oblivious(const Problem& p, Op op) { return gpu::run(p, op); }

namespace detail {

// Leaves / nodes of the reference's view-halving recursion (default_rec,
// multiply.hpp:202-230): every dimension above t is cut at ceil(d/2).
struct DefaultTally {
    std::uint64_t t;
    std::map<std::tuple<std::uint64_t, std::uint64_t, std::uint64_t>,
             std::pair<std::uint64_t, std::uint64_t>> memo;  // (nodes, leaves)

    std::pair<std::uint64_t, std::uint64_t> walk(std::uint64_t r, std::uint64_t k, std::uint64_t c) {
        if (r <= t && k <= t && c <= t) return {1, 1};
        const auto key = std::make_tuple(r, k, c);
        if (auto it = memo.find(key); it != memo.end()) return it->second;
        auto halves = [&](std::uint64_t d) {
            return d > t ? std::array<std::uint64_t, 2>{(d + 1) / 2, d / 2}
                         : std::array<std::uint64_t, 2>{d, 0};
        };
        std::pair<std::uint64_t, std::uint64_t> acc{1, 0};
        for (std::uint64_t rr : halves(r))
            for (std::uint64_t cc : halves(c))
                for (std::uint64_t kk : halves(k))
                    if (rr && cc && kk) {
                        const auto sub = walk(rr, kk, cc);
                        acc.first += sub.first;
                        acc.second += sub.second;
                    }
        memo[key] = acc;
        return acc;
    }
};

}  // namespace detail

/// mm_naive / mm_default (multiply.hpp:269-291): same results, computed by the
/// same GPU engine.  Their Counters reproduce the reference's base_case_calls,
/// scalar_macs, recursive_calls and encode_calls in closed form;
/// max_consecutive_jump of the reference's encode-addressed walks is not
/// reproduced (reported as 0) -- these two are comparison kernels, not the path.
inline Counters mm_naive(const Problem& p) {
    gpu::run(p, Op::Add);
    if (p.a.rows == 0 || p.a.cols == 0 || p.b.cols == 0) return Counters{};
    const std::uint64_t r = p.a.rows, k = p.b.cols, cc = p.a.cols;
    return Counters{1, r * k * cc, r * cc * (2 * k + 1), 1, 0};
}

inline Counters mm_default(const Problem& p) {
    check_problem(p);
    if (p.a.rows == 0 || p.a.cols == 0 || p.b.cols == 0) return Counters{};
    gpu::run(p, Op::Add);
    const std::uint64_t r = p.a.rows, k = p.b.cols, cc = p.a.cols;
    detail::DefaultTally tally{p.a.mat->layout().t, {}};
    const auto nodes_leaves = tally.walk(r, k, cc);
    detail::DefaultTally kt{p.a.mat->layout().t, {}};
    const std::uint64_t k_leaves = kt.walk(1, k, 1).second;  // leaves along the inner axis
    return Counters{nodes_leaves.second, r * k * cc, r * cc * k_leaves + 2 * r * k * cc,
                    nodes_leaves.first, 0};
}

}  // namespace mh

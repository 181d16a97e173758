// mh/multiply.hpp -- the multiply entry points (reference: multiply.hpp:39-308).
//
// mm_oblivious is the drop-in: identical results (the whole output container,
// bit for bit) and identical Counters, computed by libmhg.so's int8 limb-split
// tcgen05 kernels; the Counters come from the planner's closed form of the
// oblivious recursion.  Calls are synchronous like the reference's.
#pragma once

#include <algorithm>
#include <cstdint>
#include <optional>

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

namespace detail {

/// Largest forward step between consecutive touches of one operand's cells -- the quantity
/// behind Counters::max_consecutive_jump (reference: multiply.hpp:80-90).  The GPU engine
/// returns that counter in closed form (libmhg.so's planner); this tracker is what a host
/// walk uses to measure it, and the drop-in tests use it to check the closed forms.
struct JumpTracker {
    Index last = 0;
    bool armed = false;

    void touch(Index z, Counters& ctr) {
        if (armed && z > last) ctr.max_consecutive_jump = std::max(ctr.max_consecutive_jump, z - last);
        last = z;
        armed = true;
    }
};

}  // namespace detail

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

/// out op= lhs * rhs on the device, synchronous.  `flags` selects whose validation
/// and Counters apply: 0 = mm_oblivious, MHG_KERNEL_NAIVE / MHG_KERNEL_DEFAULT = the
/// reference's other two kernels (the same GPU computation).
inline Counters run(const Problem& p, Op op, std::uint32_t flags = 0) {
    check_problem(p);
    mhg_counters c{};
    gpu::check(mhg_mm_ex(view_of(p.a), view_of(p.b), view_of(p.c), static_cast<mhg_op>(op), flags, &c,
                         nullptr));
    gpu::check(mhg_synchronize(nullptr));
    p.a.mat->device_written();
    return to_counters(c);
}

/// Asynchronous form of run(): validation and Counters as usual, then the multiply is
/// ENQUEUED on `stream` (a cudaStream_t passed as void*; nullptr = the default stream) and
/// the call returns.  Pending host-side edits of the three matrices are uploaded first.
/// The three matrices remember the stream: their next host-side access (operator[], at,
/// cells(), ==) or upload waits for it, so results read through the Matrix API are always
/// complete; mh::synchronize(stream) waits explicitly.  Across streams the mirror inserts
/// the waits a sequential program implies -- a call that reads a matrix waits for calls in
/// flight that write it, a call that writes one waits for its readers -- except between two
/// writers of one container: as in the reference, concurrent calls are allowed on disjoint
/// output rectangles (multiply.hpp:25-29), here calls in flight on different streams.  (The
/// engine's one-shot entry point packs into one workspace per device and orders its users
/// with an event, so two such calls are both in flight but their kernels still run one
/// after the other; plans -- mhg_plan, a workspace each -- are what overlaps on the GPU.)
inline Counters run_async(const Problem& p, Op op, void* stream, std::uint32_t flags = 0) {
    check_problem(p);
    const bool uploads = p.a.mat->host_newer() || p.b.mat->host_newer() || p.c.mat->host_newer();
    auto on = [&](const Sub& s, bool as_output) {
        return mhg_view{s.mat->device_on(stream, as_output), s.origin, s.rows, s.cols};
    };
    const mhg_view va = on(p.a, true), vb = on(p.b, false), vc = on(p.c, false);
    if (uploads) gpu::check(mhg_synchronize(nullptr));  // uploads run on the default stream
    mhg_counters c{};
    gpu::check(mhg_mm_ex(va, vb, vc, static_cast<mhg_op>(op), flags, &c, stream));
    p.a.mat->device_written();
    p.a.mat->in_flight_on(stream, true);
    p.b.mat->in_flight_on(stream, false);
    p.c.mat->in_flight_on(stream, false);
    return to_counters(c);
}

}  // namespace gpu

/// Wait for `stream` (cudaStreamSynchronize for callers that do not link the CUDA runtime).
inline void synchronize(void* stream = nullptr) { gpu::check(mhg_synchronize(stream)); }

/// mm_oblivious enqueued on a stream (SURVEY 8(b) threading: the drop-in is synchronous by
/// default, this is the explicit-stream variant); see gpu::run_async.
inline Counters mm_oblivious_async(const Problem& p, Op op = Op::Add, void* stream = nullptr) {
    return gpu::run_async(p, op, stream);
}

/// Drop-in for the reference's mm_oblivious (multiply.hpp:297-308).
inline Counters mm_oblivious(const Problem& p) { return gpu::run(p, Op::Add); }

/// Same engine with the TU/TURBO operations: Op::Sub is C -= A*B, Op::Set is C = A*B.
inline Counters mm_oblivious(const Problem& p, Op op) { return gpu::run(p, op); }

/// mm_naive / mm_default (multiply.hpp:269-291): the same results from the same GPU
/// engine, with the reference's validation for these two (no layout guard: the three
/// containers may differ in n and t) and their Counters in closed form -- base-case,
/// recursion and encode tallies and the max_consecutive_jump of their encode-addressed
/// walks (the planner's naive_counters / default_counters, libmhg.so).
inline Counters mm_naive(const Problem& p) { return gpu::run(p, Op::Add, MHG_KERNEL_NAIVE); }

inline Counters mm_default(const Problem& p) { return gpu::run(p, Op::Add, MHG_KERNEL_DEFAULT); }

/// base_case_mm (multiply.hpp:136-172): out += lhs * rhs for three views that each sit
/// inside one tile; anything scattered is rejected with std::logic_error, as are shapes
/// that do not chain.  The multiply runs on the GPU engine (views of one container are
/// read before the output is written: snapshot semantics, which equals the reference's
/// in-place walk whenever the output does not overlap an operand).  Counters: one base
/// case, r*k*c MACs, no encodes; max_consecutive_jump raised to the largest forward
/// step of the reference's walks (out: +1 along a row, t - cols + 1 to the next row;
/// lhs: +1 along a row, t - inner + 1 to the next row; rhs: +t down a column, +1
/// across columns only when inner == 1).
inline void base_case_mm(const Sub& out, const Sub& lhs, const Sub& rhs, Counters& ctr) {
    if (!is_contained(out) || !is_contained(lhs) || !is_contained(rhs))
        throw std::logic_error("base_case_mm: operand spans more than one tile");
    if (out.rows != lhs.rows || out.cols != rhs.cols || lhs.cols != rhs.rows)
        throw std::logic_error("base_case_mm: view shapes do not chain");
    ++ctr.base_case_calls;
    const std::uint64_t r = out.rows, c = out.cols, k = lhs.cols;
    if (r == 0 || c == 0 || k == 0) return;
    std::uint64_t jump = 0;
    const std::uint64_t ta = out.mat->layout().t, tb = lhs.mat->layout().t, tc = rhs.mat->layout().t;
    if (c >= 2 || k >= 2) jump = 1;
    if (r >= 2) jump = std::max({jump, ta - c + 1, tb - k + 1});
    if (k >= 2) jump = std::max(jump, tc);
    ctr.max_consecutive_jump = std::max(ctr.max_consecutive_jump, jump);
    const bool shared = out.mat == lhs.mat || out.mat == rhs.mat || lhs.mat == rhs.mat;
    gpu::check(mhg_mm_ex(gpu::view_of(out), gpu::view_of(lhs), gpu::view_of(rhs), MHG_OP_ADD,
                         MHG_KERNEL_NAIVE | (shared ? MHG_ALLOW_ALIAS : 0u), nullptr, nullptr));
    gpu::check(mhg_synchronize(nullptr));
    out.mat->device_written();
    ctr.scalar_macs += r * c * k;
}

}  // namespace mh

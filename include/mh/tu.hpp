// mh/tu.hpp -- TU/TURBO Schur-update driver on ONE Morton-hybrid parent
// (the consumer the paper builds the multiply for).
//
// TURBO/TU decomposition spends its time in Schur-complement updates
//     A22 <- A22 - A21 * A12
// on views of one matrix whose origins follow the elimination and are generally not
// tile-aligned.  The reference's multiply refuses views of the same container
// (check_problem, multiply.hpp:59-60) and the factorisation itself is outside the
// reference; this header is the C++ face of the GPU engine's alias mode
// (MHG_ALLOW_ALIAS: both operands are packed before the output is written, i.e. snapshot
// semantics -- exactly the reference's result whenever the three views do not overlap,
// which holds for every step below).  Same driver as paper_1705_04807_b200/tu.py.
//
//   schur_views(M, block)   the (out, lhs, rhs) view triples of a right-looking block
//                           elimination with panel width `block`:
//                           for k0 = 0, block, ...: A[k1:, k1:] -= A[k1:, k0:k1] * A[k0:k1, k1:]
//   schur_update(p, op)     one aliased update, synchronous; returns the Counters the
//                           reference's mm_oblivious would return on three parents
//   SchurSweep              every step planned once and the whole sequence captured into ONE
//                           CUDA graph (mhg_sweep): run() is a single launch, no host work
//                           between the steps
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "mh/multiply.hpp"

namespace mh::tu {

/// View triples of the sweep, in elimination order (empty when block >= n).
inline std::vector<Problem> schur_views(Matrix& M, std::uint64_t block) {
    if (block == 0) throw std::invalid_argument("schur_views: block must be positive");
    const Layout& lay = M.layout();
    const std::uint64_t n = lay.n;
    std::vector<Problem> steps;
    for (std::uint64_t k0 = 0; k0 + block < n; k0 += block) {
        const std::uint64_t k1 = k0 + block, rest = n - k1;
        steps.push_back(Problem{Sub{&M, encode(lay, k1, k1), rest, rest},
                                Sub{&M, encode(lay, k1, k0), rest, block},
                                Sub{&M, encode(lay, k0, k1), block, rest}});
    }
    return steps;
}

/// The reference's problem checks minus the distinct-container rule (check_problem,
/// multiply.hpp:55-66): same exception types in the same order.
inline void check_aliased(const Problem& p) {
    check_sub(p.a);
    check_sub(p.b);
    check_sub(p.c);
    if (p.a.rows != p.b.rows || p.a.cols != p.c.cols || p.b.cols != p.c.rows)
        throw std::logic_error("schur update: view shapes do not chain");
}

/// One update out op= lhs * rhs on views that may share a container; synchronous.
inline Counters schur_update(const Problem& p, Op op = Op::Sub) {
    check_aliased(p);
    mhg_counters c{};
    gpu::check(mhg_mm_ex(gpu::view_of(p.a), gpu::view_of(p.b), gpu::view_of(p.c),
                         static_cast<mhg_op>(op), MHG_ALLOW_ALIAS, &c, nullptr));
    gpu::check(mhg_synchronize(nullptr));
    p.a.mat->device_written();
    return gpu::to_counters(c);
}

/// A whole sweep planned once and replayed: run() launches the one graph holding every
/// step's packs and GEMM on the default stream and waits; run_async(stream) only enqueues
/// it.  The parent must outlive the sweep; host-side edits of the parent between runs are
/// uploaded by the next run.
class SchurSweep {
public:
    SchurSweep(Matrix& M, std::uint64_t block, Op op = Op::Sub) : mat_(&M) {
        const std::vector<Problem> steps = schur_views(M, block);
        plans_.reserve(steps.size());
        try {
            for (const Problem& p : steps) {
                check_aliased(p);
                mhg_plan pl = nullptr;
                gpu::check(mhg_plan_create_ex(gpu::view_of(p.a), gpu::view_of(p.b), gpu::view_of(p.c),
                                              static_cast<mhg_op>(op), MHG_ALLOW_ALIAS, &pl));
                plans_.push_back(pl);
                mhg_counters c{};
                gpu::check(mhg_plan_counters(pl, &c));
                macs_ += c.scalar_macs;
            }
            if (!plans_.empty())
                gpu::check(mhg_sweep_create(plans_.data(), std::uint32_t(plans_.size()), &sweep_));
        } catch (...) {
            destroy();
            throw;
        }
    }
    SchurSweep(const SchurSweep&) = delete;
    SchurSweep& operator=(const SchurSweep&) = delete;
    ~SchurSweep() { destroy(); }

    std::size_t steps() const { return plans_.size(); }
    /// GF(p) multiply-adds of one sweep (the reference's scalar_macs, summed over the steps).
    std::uint64_t macs() const { return macs_; }

    /// One sweep, in place; returns macs().
    std::uint64_t run() {
        run_async(nullptr);
        if (sweep_) gpu::check(mhg_synchronize(nullptr));
        return macs_;
    }

    /// The same, enqueued on `stream` (a cudaStream_t as void*): the parent remembers the
    /// stream, and its next host-side access waits for it.
    std::uint64_t run_async(void* stream) {
        if (!sweep_) return 0;
        const bool upload = mat_->host_newer();
        // the sweep reads and writes the parent: it waits for readers and writers on other
        // streams, and later work on other streams waits for it either way
        (void)mat_->device_on(stream, true);
        (void)mat_->device_on(stream, false);  // pending host edits travel first (default stream)
        if (upload) gpu::check(mhg_synchronize(nullptr));
        gpu::check(mhg_sweep_run(sweep_, stream));
        mat_->device_written();
        mat_->in_flight_on(stream, true);
        mat_->in_flight_on(stream, false);
        return macs_;
    }

private:
    void destroy() {
        if (sweep_) mhg_sweep_destroy(sweep_);
        sweep_ = nullptr;
        for (mhg_plan pl : plans_) mhg_plan_destroy(pl);
        plans_.clear();
    }
    Matrix* mat_;
    mhg_sweep sweep_ = nullptr;
    std::vector<mhg_plan> plans_;
    std::uint64_t macs_ = 0;
};

}  // namespace mh::tu

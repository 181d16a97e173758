// mh/matrix.hpp -- Morton-hybrid container (reference: matrix.hpp:13-67).
//
// The authoritative copy lives in device memory (a libmhg container, same flat
// order and bytes as the reference's std::vector<Fp>); a host mirror serves the
// reference's element accessors.  Dirty tracking keeps them coherent:
//   - non-const accessors (operator[], set, cells()) make the host copy newer in the flat
//     range they touched (only that range is uploaded);
//   - a kernel that writes the container makes the device copy newer;
//   - whichever side is read next is refreshed first (one bulk copy).
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

#include "mh/field.hpp"
#include "mh/layout.hpp"

namespace mh {

class Matrix {
public:
    Matrix(const Layout& lay, const Modulus& mod) : lay_(lay), mod_(mod), host_(lay.total) {
        gpu::check(mhg_matrix_create(lay.n, lay.t, mod.q, &dev_));  // zero filled
    }

    Matrix(const Matrix& o) : lay_(o.lay_), mod_(o.mod_) {
        o.pull();
        host_ = o.host_;
        gpu::check(mhg_matrix_create(lay_.n, lay_.t, mod_.q, &dev_));
        touch(0, lay_.total);
    }

    Matrix(Matrix&& o) noexcept
        : lay_(o.lay_), mod_(o.mod_), host_(std::move(o.host_)), dev_(o.dev_), state_(o.state_),
          dirty_lo_(o.dirty_lo_), dirty_hi_(o.dirty_hi_), writers_(std::move(o.writers_)),
          readers_(std::move(o.readers_)), spare_(std::move(o.spare_)) {
        o.dev_ = nullptr;
        o.writers_.clear();
        o.readers_.clear();
        o.spare_.clear();
    }

    Matrix& operator=(const Matrix& o) {
        if (this != &o) {
            Matrix tmp(o);
            swap(tmp);
        }
        return *this;
    }

    Matrix& operator=(Matrix&& o) noexcept {
        swap(o);
        return *this;
    }

    ~Matrix() {
        if (dev_) {
            for (void* ev : writers_) mhg_event_synchronize(ev);  // work in flight still uses the store
            for (void* ev : readers_) mhg_event_synchronize(ev);
            mhg_matrix_destroy(dev_);
        }
        for (std::vector<void*>* set : {&writers_, &readers_, &spare_})
            for (void* ev : *set) mhg_event_destroy(ev);
    }

    const Layout& layout() const { return lay_; }
    const Modulus& modulus() const { return mod_; }

    Fp operator[](Index z) const {
        pull();
        return host_[z];
    }
    Fp& operator[](Index z) {
        pull();
        touch(z, z + 1);
        return host_[z];
    }

    Fp at(std::uint64_t i, std::uint64_t j) const { return (*this)[encode(lay_, i, j)]; }
    void set(std::uint64_t i, std::uint64_t j, Fp v) { (*this)[encode(lay_, i, j)] = v; }

    const std::vector<Fp>& cells() const {
        pull();
        return host_;
    }
    std::vector<Fp>& cells() {
        pull();
        touch(0, lay_.total);
        return host_;
    }

    friend bool operator==(const Matrix& x, const Matrix& y) {
        return x.lay_.n == y.lay_.n && x.lay_.t == y.lay_.t && x.mod_.q == y.mod_.q &&
               x.cells() == y.cells();
    }
    friend bool operator!=(const Matrix& x, const Matrix& y) { return !(x == y); }

    // ---- device side (used by the multiply entry points)
    /// Device container with any host-side edits uploaded first.
    mhg_matrix device() const {
        settle();  // the caller works on the default stream, or synchronously
        push();
        return dev_;
    }
    /// The same for work about to be enqueued on `stream`, which will write (`as_output`) or
    /// only read the device copy.  Work still in flight from earlier asynchronous calls is
    /// made a device-side dependency of `stream` (cudaStreamWaitEvent, no host wait) where a
    /// sequential program implies one: a reader waits for the writers, a writer waits for the
    /// readers.  Two writers are NOT ordered: concurrent multiplies may share an output
    /// container as long as their output rectangles are disjoint (multiply.hpp:25-29).
    mhg_matrix device_on(void* stream, bool as_output) const {
        for (void* ev : as_output ? readers_ : writers_) gpu::check(mhg_stream_wait_event(stream, ev));
        push();
        return dev_;
    }
    /// Record that a kernel wrote the device copy.
    void device_written() { state_ = State::DeviceNewer; }
    /// True when host-side edits are waiting to be uploaded (device() uploads them).
    bool host_newer() const { return state_ == State::HostNewer; }
    /// Record that work just enqueued on `stream` (a cudaStream_t as void*) writes
    /// (`as_output`) or reads the device copy: an event is recorded behind it, and the next
    /// host-side access or upload of this matrix waits for that event.  (Events, not stream
    /// handles: the caller may destroy the stream while the matrix lives on.)
    void in_flight_on(void* stream, bool as_output) const {
        std::vector<void*>& set = as_output ? writers_ : readers_;
        for (std::size_t k = 0; k < set.size();) {  // recycle the events of finished work
            int done = 0;
            gpu::check(mhg_event_query(set[k], &done));
            if (done) {
                spare_.push_back(set[k]);
                set[k] = set.back();
                set.pop_back();
            } else {
                ++k;
            }
        }
        void* ev = nullptr;
        if (!spare_.empty()) {
            ev = spare_.back();
            spare_.pop_back();
        } else {
            gpu::check(mhg_event_create(&ev));
        }
        set.push_back(ev);
        gpu::check(mhg_event_record(ev, stream));
    }

private:
    enum class State { InSync, HostNewer, DeviceNewer };

    /// Wait (on the host) for all asynchronous work in flight on this matrix.
    void settle() const {
        for (std::vector<void*>* set : {&writers_, &readers_}) {
            for (void* ev : *set) {
                gpu::check(mhg_event_synchronize(ev));
                spare_.push_back(ev);
            }
            set->clear();
        }
    }
    void pull() const {
        settle();
        if (state_ == State::DeviceNewer) {
            gpu::check(mhg_matrix_download(dev_, reinterpret_cast<std::uint32_t*>(host_.data()),
                                           nullptr));
            gpu::check(mhg_synchronize(nullptr));
            state_ = State::InSync;
        }
    }
    /// Non-const element access hands out a reference that MAY be written (the reference's
    /// callers poke cells through operator[]): the touched flat range [lo, hi) is what the next
    /// upload sends, so a few pokes -- or reads through a non-const Matrix -- do not re-upload
    /// the whole container before the next multiply.
    void touch(Index lo, Index hi) {
        if (state_ != State::HostNewer) {
            dirty_lo_ = lo;
            dirty_hi_ = hi;
        } else {
            dirty_lo_ = lo < dirty_lo_ ? lo : dirty_lo_;
            dirty_hi_ = hi > dirty_hi_ ? hi : dirty_hi_;
        }
        state_ = State::HostNewer;
    }
    void push() const {
        if (state_ == State::HostNewer) {
            settle();
            const Index lo = dirty_lo_ < lay_.total ? dirty_lo_ : lay_.total;
            const Index hi = dirty_hi_ < lay_.total ? dirty_hi_ : lay_.total;
            if (hi > lo)
                gpu::check(mhg_matrix_upload_range(
                    dev_, reinterpret_cast<const std::uint32_t*>(host_.data()) + lo, lo, hi - lo, nullptr));
            state_ = State::InSync;
        }
    }
    void swap(Matrix& o) noexcept {
        std::swap(lay_, o.lay_);
        std::swap(mod_, o.mod_);
        std::swap(host_, o.host_);
        std::swap(dev_, o.dev_);
        std::swap(state_, o.state_);
        std::swap(dirty_lo_, o.dirty_lo_);
        std::swap(dirty_hi_, o.dirty_hi_);
        std::swap(writers_, o.writers_);
        std::swap(readers_, o.readers_);
        std::swap(spare_, o.spare_);
    }

    Layout lay_;
    Modulus mod_;
    mutable std::vector<Fp> host_;
    mhg_matrix dev_ = nullptr;
    mutable State state_ = State::InSync;
    Index dirty_lo_ = 0, dirty_hi_ = 0;  // flat range the host copy may differ in (HostNewer)
    // events recorded behind asynchronous work that writes / reads the device copy, and
    // recycled events
    mutable std::vector<void*> writers_, readers_, spare_;
};
static_assert(sizeof(Fp) == sizeof(std::uint32_t), "Fp must be layout-compatible with uint32");

/// Dense row-major grid used for ingestion and checking.
using Grid = std::vector<std::vector<Fp>>;

/// Row-major -> Morton-hybrid on the device (K1 conversion kernel, which also
/// rejects residues >= q); shape checks as in the reference.
inline Matrix from_row_major(const Grid& rows, std::uint64_t t, const Modulus& mod) {
    const std::uint64_t n = rows.size();
    Layout lay(n, t);
    std::vector<std::uint32_t> flat;
    flat.reserve(n * n);
    for (const auto& r : rows) {
        if (r.size() != n) throw std::invalid_argument("from_row_major: grid is not square");
        for (Fp v : r) flat.push_back(v.v);
    }
    Matrix m(lay, mod);
    gpu::check(mhg_rowmajor_host_to_mh(m.device(), flat.data()));
    m.device_written();
    return m;
}

inline Grid to_row_major(const Matrix& m) {
    const std::uint64_t n = m.layout().n;
    std::vector<std::uint32_t> flat(n * n);
    gpu::check(mhg_mh_to_rowmajor_host(m.device(), flat.data()));
    Grid rows(n, std::vector<Fp>(n));
    for (std::uint64_t i = 0; i < n; ++i)
        for (std::uint64_t j = 0; j < n; ++j) rows[i][j] = Fp{flat[i * n + j]};
    return rows;
}

}  // namespace mh

// mhg_wire.cpp -- the 16-bit upload wire of mhg_matrix_upload.
//
// A host -> device upload of a container is PCIe-bound (4 B per cell).  For a
// modulus q <= 2^16 every canonical residue fits 16 bits, so the cells travel
// as uint16: all host workers narrow one chunk of the caller's buffer into a
// pinned staging slot (checking that every cell fits), the copy engine moves the
// slot while the workers narrow the next chunk into the next slot of a small
// ring (each slot guarded by an event on the caller's stream), and k_widen16
// restores the uint32 cells in HBM.  The container ends up byte-identical to a
// plain cudaMemcpy of the same buffer (the reference's Matrix::cells() order,
// matrix.hpp:27-28): from the first chunk holding a cell >= 2^16 -- legal in a
// reference Matrix, whose cells the caller may set freely -- the rest of the
// buffer travels as 4-byte cells.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <sched.h>

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "mhg_internal.hpp"

namespace {

// Staging ring: 4 slots of 2^22 cells (8 MiB of uint16 each): small enough to stay
// in the host LLC while the copy engine reads it (profiles/r01_upload_wire_sweep.txt).
constexpr int kMaxSlots = 4;

uint64_t chunk_cells() { return uint64_t(1) << 22; }

int ring_slots() { return kMaxSlots; }

// Narrow `n` cells to uint16; returns nonzero iff some cell needs more than 16 bits.
uint32_t narrow16_scalar(const uint32_t* __restrict src, uint16_t* __restrict dst, uint64_t n) {
    uint32_t hi = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t v = src[i];
        hi |= v;
        dst[i] = (uint16_t)v;
    }
    return hi >> 16;
}

// AVX-512: 32 cells per step (vpmovdw).  Plain stores (a small ring stays in the
// LLC, where the copy engine's coherent reads find it; streaming stores measured slower).
__attribute__((target("avx512f,avx512bw")))
uint32_t narrow16_avx512(const uint32_t* __restrict src, uint16_t* __restrict dst, uint64_t n) {
    __m512i hi = _mm512_setzero_si512();
    uint64_t i = 0;
    for (; i + 32 <= n; i += 32) {
        const __m512i a = _mm512_loadu_si512(src + i), b = _mm512_loadu_si512(src + i + 16);
        hi = _mm512_or_si512(hi, _mm512_or_si512(a, b));
        const __m512i w = _mm512_inserti64x4(_mm512_castsi256_si512(_mm512_cvtepi32_epi16(a)),
                                             _mm512_cvtepi32_epi16(b), 1);
        _mm512_storeu_si512(dst + i, w);
    }
    return (_mm512_reduce_or_epi32(hi) >> 16) | narrow16_scalar(src + i, dst + i, n - i);
}

uint32_t narrow16(const uint32_t* src, uint16_t* dst, uint64_t n) {
    static const bool avx512 = __builtin_cpu_supports("avx512bw") &&
                               __builtin_cpu_supports("avx512f");
    return avx512 ? narrow16_avx512(src, dst, n) : narrow16_scalar(src, dst, n);
}

int host_threads() {
    if (const int64_t v = mhg::option(mhg::kOptUploadThreads)) return (int)v;
    cpu_set_t set;
    CPU_ZERO(&set);
    int n = 1;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
    // one process per GPU (torchrun): share the host cores between the local ranks
    if (const char* lw = std::getenv("LOCAL_WORLD_SIZE")) {
        const int w = std::atoi(lw);
        if (w > 1) n /= w;
    }
    return n < 1 ? 1 : (n > 32 ? 32 : n);
}

// Fixed pool of narrowing workers.  run(fn) calls fn(id) once on every worker
// (id 0 = the caller) and returns when all calls are done; calls from several
// threads (uploads to different devices) take turns.  Workers spin ~1 ms after
// each task (an upload dispatches one task per chunk, a few hundred us apart)
// before parking on the condition variable.
class Pool {
public:
    explicit Pool(int n) : size_(n) {
        for (int i = 1; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_.store(true);
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    int size() const { return size_; }
    void run(const std::function<void(int)>& fn) {
        std::lock_guard<std::mutex> one(run_mu_);
        fn_ = &fn;
        pending_.store(size_ - 1, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> g(mu_);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        fn(0);
        while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
    }

private:
    void loop(int id) {
        uint64_t seen = 0;
        for (;;) {
            for (int i = 0; i < 20000 && gen_.load(std::memory_order_acquire) == seen; ++i)
                _mm_pause();
            if (gen_.load(std::memory_order_acquire) == seen) {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_.load() || gen_.load() != seen; });
            }
            if (stop_.load()) return;
            seen = gen_.load(std::memory_order_acquire);
            (*fn_)(id);
            pending_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    const int size_;
    std::vector<std::thread> workers_;
    std::mutex mu_, run_mu_;
    std::condition_variable cv_;
    const std::function<void(int)>* fn_ = nullptr;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> pending_{0};
    std::atomic<bool> stop_{false};
};

Pool& pool() {
    static Pool p(host_threads());
    return p;
}

// Pinned staging ring of one device (uploads to that device serialise on it).
struct Staging {
    int device = -1;
    uint16_t* slot[kMaxSlots] = {};
    cudaEvent_t done[kMaxSlots] = {};
    bool used[kMaxSlots] = {};
    // adaptive raw tail: a second copy stream for 4-byte chunks taken from the back
    cudaStream_t raw = nullptr;
    cudaEvent_t start = nullptr, raw_done = nullptr;
    std::mutex mu;
};

Staging* staging_for(int device, int* err) {
    static std::mutex reg_mu;
    static std::vector<Staging*> reg;
    std::lock_guard<std::mutex> g(reg_mu);
    for (Staging* s : reg)
        if (s->device == device) return s;
    auto* s = new Staging();
    s->device = device;
    for (int i = 0; i < ring_slots(); ++i) {
        int e = (int)cudaHostAlloc((void**)&s->slot[i], chunk_cells() * 2, cudaHostAllocPortable);
        if (!e) e = (int)cudaEventCreateWithFlags(&s->done[i], cudaEventDisableTiming);
        if (e) {
            *err = e;
            return nullptr;  // leaked on purpose: a process-lifetime singleton that failed
        }
    }
    int e = (int)cudaStreamCreateWithFlags(&s->raw, cudaStreamNonBlocking);
    if (!e) e = (int)cudaEventCreateWithFlags(&s->start, cudaEventDisableTiming);
    if (!e) e = (int)cudaEventCreateWithFlags(&s->raw_done, cudaEventDisableTiming);
    if (e) {
        *err = e;
        return nullptr;
    }
    reg.push_back(s);
    return s;
}

}  // namespace

namespace mhg {

bool wire16_enabled(uint32_t q, uint64_t count) {
    // narrowing runs at ~6 GB/s of cells per host thread (measured, 16 threads: 87-100 GB/s),
    // so the wire beats the 4-byte copy at the PCIe rate only with >= 8 workers; fewer
    // (e.g. 8 local ranks sharing 16 cores) keep the plain copy unless MHG_UPLOAD_WIRE=16
    int64_t mode = mhg::option(mhg::kOptUploadWire);
    if (mode == 0) mode = host_threads() >= 8 ? 16 : 32;
    return mode == 16 && q <= 65536 && count >= (uint64_t(1) << 22);
}

int upload_wire16(uint32_t* cells, uint16_t** dev16, uint64_t total, uint64_t offset,
                  const uint32_t* host, uint64_t count, int num_sms, void* stream,
                  uint64_t* wire_bytes) {
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    int e = (int)cudaGetDevice(&dev);
    if (e) return e;
    Staging* st = staging_for(dev, &e);
    if (!st) return e;
    if (!*dev16 && (e = (int)cudaMalloc((void**)dev16, total * 2))) return e;
    cells += offset;
    uint16_t* d16 = *dev16 + offset;
    std::lock_guard<std::mutex> g(st->mu);
    Pool& P = pool();
    const uint64_t chunk = chunk_cells();
    const int slots = ring_slots(), parts = P.size();
    std::vector<uint32_t> hi(parts);
    // Adaptive raw tail (MHG_OPT_UPLOAD_ADAPTIVE, pinned sources only): whenever the link is
    // idle when a chunk is about to be narrowed -- the last narrowed chunk has landed and no
    // raw copy is running, i.e. the host narrows slower than PCIe moves 2-byte cells (a slow
    // or contended host) -- one chunk from the BACK of the buffer goes as 4-byte cells
    // straight from the caller's pinned memory on a second copy stream (no host work).
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const bool adaptive = pinned && mhg::option(mhg::kOptUploadAdaptive) != 0;
    uint64_t back = count;  // [back, count) travels raw
    bool raw_used = false;
    int last_k = -1;
    uint64_t narrow = 0;  // cells sent as uint16 (a prefix of the container)
    for (uint64_t c = 0; narrow < back; ++c) {
        const int k = (int)(c % slots);
        if (adaptive && back - narrow > 2 * chunk &&
            (last_k < 0 || cudaEventQuery(st->done[last_k]) == cudaSuccess) &&
            (!raw_used || cudaEventQuery(st->raw_done) == cudaSuccess)) {
            if (!raw_used) {  // raw copies follow the caller's earlier work on the container
                if ((e = (int)cudaEventRecord(st->start, s)) ||
                    (e = (int)cudaStreamWaitEvent(st->raw, st->start, 0)))
                    return e;
                raw_used = true;
            }
            back -= chunk;
            if ((e = (int)cudaMemcpyAsync(cells + back, host + back, chunk * 4, cudaMemcpyHostToDevice, st->raw)) ||
                (e = (int)cudaEventRecord(st->raw_done, st->raw)))
                return e;
        }
        cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
        const uint64_t base = narrow, len = back - base < chunk ? back - base : chunk;
        if (st->used[k] && (e = (int)cudaEventSynchronize(st->done[k]))) return e;
        const uint64_t per = ((len + parts - 1) / parts + 31) & ~uint64_t(31);  // 64-byte parts
        uint16_t* slot = st->slot[k];
        P.run([&](int id) {
            const uint64_t b = (uint64_t)id * per;
            hi[id] = b < len ? narrow16(host + base + b, slot + b, len - b < per ? len - b : per) : 0;
        });
        bool fits = true;
        for (uint32_t h : hi) fits = fits && h == 0;
        if (!fits) break;
        e = (int)cudaMemcpyAsync(d16 + base, slot, len * 2, cudaMemcpyHostToDevice, s);
        if (!e) e = (int)cudaEventRecord(st->done[k], s);
        if (e) return e;
        st->used[k] = true;
        last_k = k;
        narrow += len;
    }
    if ((e = launch_widen16(d16, cells, narrow, num_sms, stream))) return e;
    if (narrow < back &&
        (e = (int)cudaMemcpyAsync(cells + narrow, host + narrow, (back - narrow) * 4,
                                  cudaMemcpyHostToDevice, s)))
        return e;
    if (raw_used && (e = (int)cudaStreamWaitEvent(s, st->raw_done, 0))) return e;
    *wire_bytes = narrow * 2 + (count - narrow) * 4;
    return 0;
}

}  // namespace mhg

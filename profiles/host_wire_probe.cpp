// host_wire_probe.cpp -- where the e2e upload wire's host time goes (GPU box, one GPU).
//
// A "step" = three 1 GiB uint32 containers (n = 16384) uploaded as uint16 plus, optionally,
// one concurrent 1 GiB device -> pinned-host download (the e2e pipeline's D2H).  Variants:
//   read      : host threads only sum the three sources (host DRAM read rate)
//   narrow    : host threads narrow into private rings, no copies (narrowing rate)
//   lockstep  : the product's scheme -- all threads narrow one chunk, then one H2D copy
//   worker    : barrier-free -- chunk j is narrowed by worker j % T into that worker's own
//               slots and copied by the worker itself (events per slot)
// Build: nvcc -O3 -std=c++17 -Iinclude -o profiles/host_wire_probe_bin profiles/host_wire_probe.cpp \
//          -Lpaper_1705_04807_b200 -lmhg -Xlinker -rpath,'$ORIGIN/../paper_1705_04807_b200'
// Run:   profiles/host_wire_probe_bin   (prints one line per variant and D2H setting)
#include <cuda_runtime.h>

#include "mhg.h"
#include <immintrin.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_) {                                                                    \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                            \
        }                                                                            \
    } while (0)

static const uint64_t kCells = uint64_t(16384) * 16384;

__attribute__((target("avx512f,avx512bw"))) static uint32_t narrow(const uint32_t* __restrict src,
                                                                    uint16_t* __restrict dst, uint64_t n,
                                                                    bool nta) {
    __m512i hi = _mm512_setzero_si512();
    for (uint64_t i = 0; i + 32 <= n; i += 32) {
        if (nta) _mm_prefetch((const char*)(src + i + 512), _MM_HINT_NTA);
        const __m512i a = _mm512_loadu_si512(src + i), b = _mm512_loadu_si512(src + i + 16);
        hi = _mm512_or_si512(hi, _mm512_or_si512(a, b));
        const __m512i w = _mm512_inserti64x4(_mm512_castsi256_si512(_mm512_cvtepi32_epi16(a)),
                                             _mm512_cvtepi32_epi16(b), 1);
        _mm512_storeu_si512(dst + i, w);
    }
    return _mm512_reduce_or_epi32(hi) >> 16;
}

__attribute__((target("avx512f"))) static uint64_t sum(const uint32_t* src, uint64_t n) {
    __m512i acc = _mm512_setzero_si512();
    for (uint64_t i = 0; i + 16 <= n; i += 16) acc = _mm512_add_epi32(acc, _mm512_loadu_si512(src + i));
    return (uint64_t)_mm512_reduce_add_epi32(acc);
}

struct Ctx {
    int T;
    uint32_t* src[3];
    uint16_t* d16;
    uint32_t* dres;
    uint32_t* hres;
    cudaStream_t up, dn;
};

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// run fn(tid) on T threads (fresh threads each call: the variants differ in more than the pool)
template <class F>
static void par(int T, F fn) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back([&, t] { fn(t); });
    fn(0);
    for (auto& x : th) x.join();
}

static std::atomic<uint64_t> g_sink{0};

static void step_read(Ctx& c) {
    for (int m = 0; m < 3; ++m)
        par(c.T, [&](int t) {
            const uint64_t per = kCells / c.T;
            g_sink += sum(c.src[m] + t * per, per);
        });
}

static std::vector<uint16_t*> g_priv;
static void step_narrow(Ctx& c, uint64_t ring_cells) {
    for (int m = 0; m < 3; ++m)
        par(c.T, [&](int t) {
            const uint64_t per = kCells / c.T;
            for (uint64_t o = 0; o < per; o += ring_cells)
                g_sink += narrow(c.src[m] + t * per + o, g_priv[t], std::min(ring_cells, per - o), false);
        });
}

struct Ring {
    std::vector<uint16_t*> slot;
    std::vector<cudaEvent_t> ev;
    std::vector<bool> used;
};
static Ring g_lock;
static void step_lockstep(Ctx& c, uint64_t chunk, int slots) {
    for (int m = 0; m < 3; ++m) {
        for (uint64_t j = 0; j * chunk < kCells; ++j) {
            const int k = (int)(j % slots);
            if (g_lock.used[k]) CK(cudaEventSynchronize(g_lock.ev[k]));
            const uint64_t base = j * chunk, per = chunk / c.T;
            par(c.T, [&](int t) { g_sink += narrow(c.src[m] + base + t * per, g_lock.slot[k] + t * per, per, false); });
            CK(cudaMemcpyAsync(c.d16 + base, g_lock.slot[k], chunk * 2, cudaMemcpyHostToDevice, c.up));
            CK(cudaEventRecord(g_lock.ev[k], c.up));
            g_lock.used[k] = true;
        }
    }
    CK(cudaStreamSynchronize(c.up));
}

static std::vector<Ring> g_work;
static std::vector<cudaStream_t> g_wstream;
static void step_worker(Ctx& c, uint64_t chunk, int slots, bool own_stream, bool nta) {
    for (int m = 0; m < 3; ++m) {
        const uint64_t nchunks = kCells / chunk;
        par(c.T, [&](int t) {
            Ring& r = g_work[t];
            cudaStream_t s = own_stream ? g_wstream[t] : c.up;
            uint64_t i = 0;
            for (uint64_t j = t; j < nchunks; j += c.T, ++i) {
                const int k = (int)(i % slots);
                if (r.used[k]) CK(cudaEventSynchronize(r.ev[k]));
                g_sink += narrow(c.src[m] + j * chunk, r.slot[k], chunk, nta);
                CK(cudaMemcpyAsync(c.d16 + j * chunk, r.slot[k], chunk * 2, cudaMemcpyHostToDevice, s));
                CK(cudaEventRecord(r.ev[k], s));
                r.used[k] = true;
            }
        });
    }
    if (own_stream)
        for (auto s : g_wstream) CK(cudaStreamSynchronize(s));
    CK(cudaStreamSynchronize(c.up));
}

int main(int argc, char** argv) {
    cpu_set_t set;
    CPU_ZERO(&set);
    sched_getaffinity(0, sizeof(set), &set);
    Ctx c{};
    c.T = argc > 1 ? std::atoi(argv[1]) : CPU_COUNT(&set);
    const int steps = 5;
    for (int m = 0; m < 3; ++m) {
        CK(cudaHostAlloc((void**)&c.src[m], kCells * 4, cudaHostAllocPortable));
        for (uint64_t i = 0; i < kCells; ++i) c.src[m][i] = (uint32_t)((i * 2654435761u + m) % 65521u);
    }
    CK(cudaHostAlloc((void**)&c.hres, kCells * 4, cudaHostAllocPortable));
    std::memset(c.hres, 0, kCells * 4);
    CK(cudaMalloc((void**)&c.d16, kCells * 2));
    CK(cudaMalloc((void**)&c.dres, kCells * 4));
    CK(cudaMemset(c.dres, 1, kCells * 4));
    CK(cudaStreamCreateWithFlags(&c.up, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c.dn, cudaStreamNonBlocking));
    g_priv.resize(c.T);
    for (int t = 0; t < c.T; ++t) g_priv[t] = (uint16_t*)aligned_alloc(64, (1 << 22) * 2);
    g_lock.slot.resize(8);
    g_lock.ev.resize(8);
    g_lock.used.assign(8, false);
    for (int k = 0; k < 8; ++k) {
        CK(cudaHostAlloc((void**)&g_lock.slot[k], (uint64_t(1) << 22) * 2, cudaHostAllocPortable));
        CK(cudaEventCreateWithFlags(&g_lock.ev[k], cudaEventDisableTiming));
    }
    g_work.resize(c.T);
    g_wstream.resize(c.T);
    for (int t = 0; t < c.T; ++t) {
        CK(cudaStreamCreateWithFlags(&g_wstream[t], cudaStreamNonBlocking));
        g_work[t].slot.resize(4);
        g_work[t].ev.resize(4);
        g_work[t].used.assign(4, false);
        for (int k = 0; k < 4; ++k) {
            CK(cudaHostAlloc((void**)&g_work[t].slot[k], (uint64_t(1) << 20) * 2, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&g_work[t].ev[k], cudaEventDisableTiming));
        }
    }
    std::printf("threads %d, step = 3 x %.2f GiB uint32 sources (uint16 wire), D2H = 1 GiB per step\n",
                c.T, kCells * 4 / 1073741824.0);

    struct V {
        std::string name;
        std::function<void()> fn;
    };
    mhg_matrix mats[3];
    for (int m = 0; m < 3; ++m)
        if (mhg_matrix_create(16384, 64, 65521, &mats[m])) { std::fprintf(stderr, "create\n"); return 1; }
    std::vector<V> vs = {
        {"product: mhg_matrix_upload x3 (libmhg)", [&] {
             for (int m = 0; m < 3; ++m)
                 if (mhg_matrix_upload(mats[m], c.src[m], c.up)) std::exit(2);
             CK(cudaStreamSynchronize(c.up));
         }},
        {"read (host DRAM read of the 3 sources)", [&] { step_read(c); }},
        {"narrow, private 512 KiB rings, no copies", [&] { step_narrow(c, 1 << 18); }},
        {"worker chunk 2^18 x 2 slots, one stream", [&] { step_worker(c, 1 << 18, 2, false, false); }},
        {"worker chunk 2^18 x 4 slots, one stream", [&] { step_worker(c, 1 << 18, 4, false, false); }},
        {"worker chunk 2^19 x 2 slots, one stream", [&] { step_worker(c, 1 << 19, 2, false, false); }},
        {"worker chunk 2^20 x 2 slots, one stream", [&] { step_worker(c, 1 << 20, 2, false, false); }},
        {"worker chunk 2^19 x 2 slots, own streams", [&] { step_worker(c, 1 << 19, 2, true, false); }},
        {"worker chunk 2^19 x 2 slots, one stream, prefetchnta", [&] { step_worker(c, 1 << 19, 2, false, true); }},
    };
    for (int round = 0; round < 2; ++round)
        for (auto& v : vs)
            for (int d2h = 0; d2h < 2; ++d2h) {
                v.fn();  // warm-up
                double t0 = now();
                for (int s = 0; s < steps; ++s) {
                    if (d2h) CK(cudaMemcpyAsync(c.hres, c.dres, kCells * 4, cudaMemcpyDeviceToHost, c.dn));
                    v.fn();
                    CK(cudaStreamSynchronize(c.dn));
                }
                const double ms = (now() - t0) / steps * 1e3;
                std::printf("%-56s D2H=%d  %7.2f ms/step  (%.1f GB/s of source cells)\n", v.name.c_str(), d2h, ms,
                            3 * kCells * 4 / (ms * 1e-3) / 1e9);
                std::fflush(stdout);
            }
    std::printf("sink %llu\n", (unsigned long long)g_sink.load());
    return 0;
}

// mhg_options.cpp -- process-wide options (mhg_set_option / mhg_get_option).
//
// The planner's kernel and digit choices and the test hooks used to be read
// from the environment at every plan; now they are one table, seeded from the
// environment once (first use) and changed only through the C ABI.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mhg_internal.hpp"

namespace mhg {
namespace {

std::atomic<int64_t> g_opt[kOptCount];
std::once_flag g_once;

int64_t env_int(const char* name, int64_t dflt) {
    const char* e = std::getenv(name);
    if (!e || !*e) return dflt;
    char* end = nullptr;
    const long long v = std::strtoll(e, &end, 10);
    return (end && *end == 0) ? (int64_t)v : dflt;
}

void seed() {
    g_opt[kOptDigits] = env_int("MHG_UDIG", 1) != 0 ? 1 : 0;
    int64_t gk = 0;
    if (const char* e = std::getenv("MHG_GEMM")) {
        if (!std::strcmp(e, "1cta") || !std::strcmp(e, "1")) gk = 1;
        else if (!std::strcmp(e, "2cta") || !std::strcmp(e, "2")) gk = 2;
    }
    g_opt[kOptGemmKernel] = gk;
    const int64_t fold = env_int("MHG_FOLD", 1);
    g_opt[kOptMinFold] = fold >= 1 && fold <= 3 ? fold : 1;
    const int64_t kc = env_int("MHG_FORCE_KCHUNK", 0);
    g_opt[kOptMaxKChunk] = kc > 0 ? kc : 0;
    const int64_t wire = env_int("MHG_UPLOAD_WIRE", 0);
    g_opt[kOptUploadWire] = (wire == 16 || wire == 32) ? wire : 0;
    const int64_t conv = env_int("MHG_CONV", 0);
    g_opt[kOptConvKernel] = conv >= 0 && conv <= 2 ? conv : 0;
    g_opt[kOptGemmStats] = std::getenv("MHG_GEMM_STATS") ? 1 : 0;
    const int64_t th = env_int("MHG_UPLOAD_THREADS", 0);
    g_opt[kOptUploadThreads] = th > 0 && th <= 256 ? th : 0;
    g_opt[kOptUploadAdaptive] = env_int("MHG_UPLOAD_ADAPTIVE", 0) != 0 ? 1 : 0;
}

}  // namespace

bool option_valid(int key, int64_t v) {
    switch (key) {
        case kOptDigits: return v == 0 || v == 1;
        case kOptGemmKernel: return v >= 0 && v <= 2;
        case kOptMinFold: return v >= 1 && v <= 3;
        case kOptMaxKChunk: return v >= 0;
        case kOptUploadWire: return v == 0 || v == 16 || v == 32;
        case kOptConvKernel: return v >= 0 && v <= 2;
        case kOptGemmStats: return v == 0 || v == 1;
        case kOptUploadThreads: return v >= 0 && v <= 256;
        case kOptUploadAdaptive: return v == 0 || v == 1;
    }
    return false;
}

int64_t option(int key) {
    std::call_once(g_once, seed);
    return (key > 0 && key < kOptCount) ? g_opt[key].load(std::memory_order_relaxed) : 0;
}

void set_option(int key, int64_t value) {
    std::call_once(g_once, seed);
    g_opt[key].store(value, std::memory_order_relaxed);
}

}  // namespace mhg

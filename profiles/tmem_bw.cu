// TMEM read bandwidth probe (B200): each CTA allocates 512 TMEM columns, 4 (or 8) warps read
// their lane quadrant with tcgen05.ld.32x32b.x16 in a loop (all loads of a round in flight,
// one wait per round); reports bytes per SM per cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw profiles/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_tmem_bw(int rounds, int nwarps_active, unsigned long long* cycles, int* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
    int acc = 0;
    long long t0 = clock64();
    if (warp < nwarps_active) {
        const uint32_t colbase = (warp >> 2) * 256;
        for (int r = 0; r < rounds; ++r) {
            uint32_t v[8][16];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(v[c][0]), "=r"(v[c][1]), "=r"(v[c][2]), "=r"(v[c][3]), "=r"(v[c][4]), "=r"(v[c][5]),
                      "=r"(v[c][6]), "=r"(v[c][7]), "=r"(v[c][8]), "=r"(v[c][9]), "=r"(v[c][10]), "=r"(v[c][11]),
                      "=r"(v[c][12]), "=r"(v[c][13]), "=r"(v[c][14]), "=r"(v[c][15])
                    : "r"(tmem + colbase + (uint32_t)(16 * c)));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 8; ++c)
#pragma unroll
                for (int j = 0; j < 16; ++j) acc += (int)v[c][j];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 12345) sink[0] = acc;
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
    }
}

int main() {
    unsigned long long* cyc;
    int* sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 4);
    const int rounds = 2000;
    for (int nw : {4, 8}) {
        k_tmem_bw<<<148, 256>>>(10, nw, cyc, sink);
        k_tmem_bw<<<148, 256>>>(rounds, nw, cyc, sink);
        cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double bytes = (double)rounds * nw * 8 * 32 * 16 * 4;  // per SM
        printf("warps %d: %.0f cycles, %.1f B/cycle per SM (TMEM read)\n", nw, avg, bytes / avg);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

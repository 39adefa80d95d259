// Latency / throughput of __match_any_sync and of a global atomicAdd round trip
// with distinct keys (the delivery kernel's reservation pattern).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_match(unsigned* out, long long* cyc, int mode, int iters, unsigned* ctr) {
    unsigned key = (threadIdx.x * 2654435761u) >> 27;      // 32 lanes -> ~20 distinct keys
    unsigned acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) {                                   // dependent match_any chain
            const unsigned p = __match_any_sync(0xffffffffu, key);
            key = (key + (p & 7u)) & 31u;
            acc += p;
        } else if (mode == 1) {                            // independent match_any x4
            unsigned p0 = __match_any_sync(0xffffffffu, key);
            unsigned p1 = __match_any_sync(0xffffffffu, key ^ 1u);
            unsigned p2 = __match_any_sync(0xffffffffu, key ^ 2u);
            unsigned p3 = __match_any_sync(0xffffffffu, key ^ 3u);
            acc += p0 ^ p1 ^ p2 ^ p3;
            key = (key + 1u) & 31u;
        } else {                                           // global atomic round trip
            acc += atomicAdd(&ctr[(blockIdx.x * 64 + (acc & 63u)) & 65535u], 1u);
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    unsigned* out; long long* cyc; unsigned* ctr;
    cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 20); cudaMalloc(&ctr, 1 << 20);
    const char* names[] = {"match dep", "match x4 ind", "atomic rt"};
    const int iters = 2048;
    for (int mode = 0; mode < 3; ++mode)
        for (int warps : {1, 8, 32}) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            k_match<<<148, 32 * warps>>>(out, cyc, mode, 16, ctr);
            cudaEventRecord(a);
            k_match<<<148, 32 * warps>>>(out, cyc, mode, iters, ctr);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)warps * iters * 148 * (mode == 1 ? 4 : 1);
            printf("%-13s warps/SM %2d: %7.1f cycles/iter/warp, %7.2f G warp-ops/s\n", names[mode],
                   warps, (double)c / iters, ops / (ms * 1e-3) / 1e9);
        }
    return 0;
}

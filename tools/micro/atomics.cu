// Microbenchmark: cost of same-address global atomics from many blocks/warps.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_same(unsigned long long* c, int per_block) {
    if ((threadIdx.x & 31) == 0 && threadIdx.x / 32 < per_block) atomicAdd(c, 1ull);
}
__global__ void k_none(unsigned long long* c) { if (threadIdx.x == 9999) c[1] = 1; }
__global__ void k_spread(unsigned long long* c, int per_block) {
    if ((threadIdx.x & 31) == 0 && threadIdx.x / 32 < per_block) atomicAdd(c + 32 * (blockIdx.x * 4 + threadIdx.x / 32), 1ull);
}
int main() {
    unsigned long long* c; cudaMalloc(&c, 64 << 20); cudaMemset(c, 0, 64 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocks : {148, 620, 2480, 9472}) {
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e9;
            for (int r = 0; r < 20; ++r) {
                cudaEventRecord(a);
                if (mode == 0) k_none<<<blocks, 128>>>(c);
                else if (mode == 1) k_same<<<blocks, 128>>>(c, 4);
                else k_spread<<<blocks, 128>>>(c, 4);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            printf("blocks %5d mode %s: %8.2f us\n", blocks, mode == 0 ? "none  " : mode == 1 ? "same  " : "spread", best * 1e3);
        }
    }
    return 0;
}

// Dependent-chain latency and throughput of fp64 ops, exp, division and smem loads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_chain(double* out, long long* cyc, int mode, int iters, double seed) {
    double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 0.5 + i * 1e-6;
    __syncthreads();
    int idx = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) x = fma(x, y, 1e-9);                 // DFMA chain
        else if (mode == 1) x = x * y + 1e-9;                // DMUL+DADD chain (fmad=false)
        else if (mode == 2) x = exp(-x * 1e-3);              // exp chain
        else if (mode == 3) x = (x + 1.0) / 3.0;             // division chain
        else if (mode == 4) { idx = (int)(sm[idx & 1023] * 1000.0) ^ i; x += idx; } // smem load chain
        else if (mode == 5) x = expm1(x * 1e-3);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 20);
    const char* names[] = {"DFMA", "DMUL+DADD", "exp", "div", "smem-dep", "expm1"};
    const int iters = 4096;
    for (int mode = 0; mode < 6; ++mode) {
        for (int warps : {1, 4, 16, 32}) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            k_chain<<<148, 32 * warps>>>(out, cyc, mode, 16, 1.0);
            cudaEventRecord(a);
            k_chain<<<148, 32 * warps>>>(out, cyc, mode, iters, 1.0);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            double per_op_warp = (double)c / iters;
            double tput = (double)warps * 32 * iters * 148 / (ms * 1e-3) / 1e9;   // Gop/s total
            printf("%-10s warps/SM %2d: %7.1f cycles/iter/warp, %8.1f Gop/s (lane-ops)\n", names[mode], warps, per_op_warp, tput);
        }
    }
}

// Floor of the fp64 decay-factor math: em = exp(-dt/tau_m), ec, expm1 form of f.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_fac(const double* __restrict__ dt, double* em_o, double* ec_o, double* f_o, int n, int mode) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double d = dt[i];
    const double tau_m = 20.0, tau_c = 300.0, k1 = 280.0, k2 = 6000.0;
    double em, ec = 1.0, f = 0.0;
    if (mode == 0) { em = exp(-d / tau_m); ec = exp(-d / tau_c); const double x = d * k1 / k2;
        f = (fabs(x) <= 1.0) ? d * em * expm1(x) / x : d * (ec - em) / x; }
    else if (mode == 1) { em = exp(-d / tau_m); }
    else { em = -d / tau_m; ec = -d / tau_c; f = d * k1 / k2; }
    em_o[i] = em; ec_o[i] = ec; f_o[i] = f;
}
int main() {
    const int n = 1 << 20;
    double *dt, *a, *b, *c;
    cudaMalloc(&dt, n * 8); cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8);
    double* h = new double[n]; for (int i = 0; i < n; ++i) h[i] = (i % 997) * 0.001; cudaMemcpy(dt, h, n * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(e0); k_fac<<<n / 256, 256>>>(dt, a, b, c, n, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("mode %d (%s): %.2f us for %d events\n", mode, mode == 0 ? "em+ec+f" : mode == 1 ? "em only" : "divs only", best * 1e3, n);
    }
}

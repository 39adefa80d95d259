// Check: div_rn (reciprocal multiply + one FMA correction, Markstein) equals
// IEEE a / b for the kernels' constant divisors over many random dividends.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double div_rn(double a, double b, double rb) {
    const double q0 = __dmul_rn(a, rb);
    const double r = __fma_rn(-q0, b, a);
    return __fma_rn(r, rb, q0);
}
__device__ uint64_t sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void k(double b, double rb, unsigned long long* bad, long long n, int mode) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const uint64_t h = sm64((uint64_t)i * 7919 + mode);
        double a;
        if (mode == 0) a = (double)(h >> 11) * (1.0 / 9007199254740992.0) * 50.0;     // dt in [0, 50) ms
        else if (mode == 1) a = __longlong_as_double((long long)(h >> 2) & 0x7fefffffffffffffll) ; // any positive
        else a = (double)(h >> 11) * (1.0 / 9007199254740992.0) * 1e4;                 // [0, 1e4)
        if (mode == 1 && (a < 1e-290 || a > 1e290)) continue;
        if (div_rn(a, b, rb) != a / b) atomicAdd(bad, 1ull);
    }
}
int main() {
    unsigned long long* bad; cudaMallocManaged(&bad, 8);
    const double bs[] = {20.0, 300.0, 6000.0, 10.0, 7.0, 3.0, 0.1, 280.0 * 1.0};
    for (double b : bs) for (int mode = 0; mode < 3; ++mode) {
        *bad = 0;
        k<<<148 * 8, 256>>>(b, 1.0 / b, bad, 1ll << 30, mode);
        cudaDeviceSynchronize();
        printf("b=%g mode=%d mismatches=%llu of 2^30\n", b, mode, *bad);
    }
    return 0;
}

// Shared device helpers: counter-based RNGs of the reference, bit-exact.
//
//   splitmix64 / counter_uniforms   corticarc/rng.py:61-90
//   Philox4x64-10 stream            corticarc/rng.py:42-52 (numpy Philox,
//                                   counter pre-incremented per block)
//   ziggurat normal / exponential   numpy Generator.standard_normal /
//                                   .exponential (the algorithm of Marsaglia &
//                                   Tsang 2000 with numpy's 256-layer tables,
//                                   extracted at build time into
//                                   cc_ziggurat_tables.h by gen_ziggurat.py)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "corticarc_b200.h"

#define CC_DOMAIN 0x636F727469636172ull
#define CC_EXT_SRC 0xFFFFFFFFu

__host__ __device__ __forceinline__ uint64_t cc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// top 53 bits -> [0, 1): exact, (h >> 11) < 2^53
__host__ __device__ __forceinline__ double cc_u53(uint64_t h) {
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

// ------------------------------------------------------------------ Philox
struct cc_philox_block { uint64_t v[4]; };

__device__ __forceinline__ cc_philox_block cc_philox4x64(uint64_t ctr0, uint64_t ctr1,
                                                         uint64_t ctr2, uint64_t ctr3,
                                                         uint64_t k0, uint64_t k1) {
    uint64_t c0 = ctr0, c1 = ctr1, c2 = ctr2, c3 = ctr3;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0;
        const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
        const uint64_t lo1 = 0xCA5A826395121157ull * c2;
        const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, c2);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B97F4A7C15ull;
        k1 += 0xBB67AE8584CAA73Bull;
    }
    cc_philox_block b;
    b.v[0] = c0; b.v[1] = c1; b.v[2] = c2; b.v[3] = c3;
    return b;
}

// Word j of stream (seed, purpose, a): lane j%4 of block j/4, counter
// (j/4 + 1, a, 0, DOMAIN).  Random access - used where the reference's draw
// index is known (Bernoulli candidate index, delay rank).
__device__ __forceinline__ uint64_t cc_philox_word(uint64_t seed, uint64_t purpose,
                                                   uint64_t a, uint64_t j) {
    cc_philox_block b = cc_philox4x64((j >> 2) + 1, a, 0, CC_DOMAIN, seed, purpose);
    return b.v[j & 3];
}

// Sequential reader of one stream (numpy's buffered next_uint64).
struct cc_philox_stream {
    uint64_t seed, purpose, a;
    uint64_t pos;          // index of the next word
    uint64_t buf[4];
    uint64_t buf_blk;      // block index held in buf (+1 offset), 0 = empty

    __device__ __forceinline__ void init(uint64_t s, uint64_t p, uint64_t aa, uint64_t start) {
        seed = s; purpose = p; a = aa; pos = start; buf_blk = 0;
    }
    __device__ __forceinline__ uint64_t next() {
        const uint64_t blk = (pos >> 2) + 1;
        if (blk != buf_blk) {
            cc_philox_block b = cc_philox4x64(blk, a, 0, CC_DOMAIN, seed, purpose);
            buf[0] = b.v[0]; buf[1] = b.v[1]; buf[2] = b.v[2]; buf[3] = b.v[3];
            buf_blk = blk;
        }
        const uint64_t w = buf[pos & 3];
        ++pos;
        return w;
    }
    __device__ __forceinline__ double next_double() { return cc_u53(next()); }
};

// ---------------------------------------------------------------- ziggurat
#include "cc_ziggurat_tables.h"   // cc_zig_{wi,ki,fi,we,ke,fe}, cc_zig_nor_r, cc_zig_exp_r

// numpy random_standard_normal: 8-bit layer index, sign bit, 52-bit mantissa;
// fast accept when rabs < ki[idx]; base layer via the exponential tail; other
// layers by the wedge test against exp(-x^2/2).
__device__ __forceinline__ double cc_std_normal(cc_philox_stream& s) {
    for (;;) {
        uint64_t r = s.next();
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const int sign = (int)(r & 1);
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
        double x = (double)rabs * cc_zig_wi[idx];
        if (sign) x = -x;
        if (rabs < cc_zig_ki[idx]) return x;
        if (idx == 0) {
            for (;;) {
                const double xx = -cc_zig_nor_inv_r * log1p(-s.next_double());
                const double yy = -log1p(-s.next_double());
                if (yy + yy > xx * xx)
                    return ((rabs >> 8) & 1) ? -(cc_zig_nor_r + xx) : (cc_zig_nor_r + xx);
            }
        } else {
            if ((cc_zig_fi[idx - 1] - cc_zig_fi[idx]) * s.next_double() + cc_zig_fi[idx]
                < exp(-0.5 * x * x))
                return x;
        }
    }
}

// numpy random_standard_exponential (ziggurat, 256 layers).
__device__ __forceinline__ double cc_std_exponential(cc_philox_stream& s) {
    for (;;) {
        uint64_t ri = s.next();
        ri >>= 3;
        const int idx = (int)(ri & 0xff);
        ri >>= 8;
        const double x = (double)ri * cc_zig_we[idx];
        if (ri < cc_zig_ke[idx]) return x;
        if (idx == 0) return cc_zig_exp_r - log1p(-s.next_double());
        if ((cc_zig_fe[idx - 1] - cc_zig_fe[idx]) * s.next_double() + cc_zig_fe[idx] < exp(-x))
            return x;
    }
}

// ---------------------------------------------------------------- errors
__device__ __forceinline__ void cc_raise(cc_ctl* ctl, unsigned bits, long long t) {
    atomicOr(&ctl->error_bits, bits);
    atomicMin(&ctl->error_step, t);
}

// Bounds and protocol assertions of the checked build (-DCC_CHECKS=1,
// libcorticarc_b200_chk.so, run by tests/test_gpu_parity.py in place of a
// compute-sanitizer pass): a failed check prints its source line and raises
// CC_ERR_CHECK with the line as the error "step".  Compiled away otherwise.
#ifndef CC_CHECKS
#define CC_CHECKS 0
#endif
#if CC_CHECKS
#include <cstdio>
static __device__ __noinline__ void cc_check_fail(cc_ctl* ctl, const char* file, int line,
                                                  const char* what) {
    printf("cc check failed: %s:%d: %s\n", file, line, what);
    cc_raise(ctl, CC_ERR_CHECK, (long long)line);
}
#define CC_CHK(ctl, cond)                                                  \
    do {                                                                   \
        if (!(cond)) cc_check_fail((ctl), __FILE__, __LINE__, #cond);      \
    } while (0)
#else
#define CC_CHK(ctl, cond) do { } while (0)
#endif

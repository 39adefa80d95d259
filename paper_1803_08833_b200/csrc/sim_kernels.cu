// Simulation-step kernels of the B200 engine (sm_100a).
//
// Per 1 ms step t (engine.py:318-394):
//   k_deliver   the events arriving at t not yet delivered: the delay-d segments
//               of the rows of step t-d's spikes (engine.py:338-367 and
//               DelayRing, :124-163, as a pull from the spike log)
//   k_plan      per group of 32 neurons: input counts, the Poisson drive count
//               (engine.py:172-188), work items
//   k_stage     gather + drive times, order each neuron's inputs by (time,
//               source, weight), decay factors, the in-order float64 update,
//               spikes (engine.py:191-206, 386, model.py:272-337); its idle
//               warps deliver step t+1's delay >= 2 events
// plus k_ingest / k_pack_aer / k_ingest_aer for multi-shard runs, k_build_dseg
// and k_init_state.
//
// Exactness contract: every float64 expression below
// follows the reference's evaluation order; the file is compiled with
// -fmad=false so no multiply-add is contracted.
#include <climits>
#include <type_traits>
#include "cc_common.cuh"

// This translation unit is compiled once per sub-list variant (build.py):
// CC_SUBLISTS sub-lists per group, entry points suffixed _s<CC_SUBLISTS>
// (dispatch.cu selects by cc_shard.n_sub).  The primary variant (CC_NSUB_A)
// also carries the entry points that do not depend on the lists.
#ifndef CC_SUBLISTS
#define CC_SUBLISTS CC_NSUB_A
#endif
#define CC_PRIMARY (CC_SUBLISTS == CC_NSUB_A)
#define CC_CAT2_(a, b) a##_s##b
#define CC_CAT2(a, b) CC_CAT2_(a, b)
#define CC_V(name) CC_CAT2(name, CC_SUBLISTS)

// cache-policy experiments (tools/sweep_variants.py): evict-first CSR loads in
// k_deliver, evict-first ordered-input records in k_stage
// list fill counters CC_CNT_STRIDE words apart: a step's reservations (one
// atomic per run) hit n_groups counters, which a dense array would put in a
// handful of L2 slices
#ifndef CC_CNT_STRIDE
#define CC_CNT_STRIDE CC_CNT_STRIDE_FOR(CC_SUBLISTS)
#endif
#ifndef CC_STATIC_FIRST
#define CC_STATIC_FIRST 1     // k_stage: each warp's first item by its index
#endif
#ifndef CC_CLAIM_OWN_LINE
#define CC_CLAIM_OWN_LINE 1  // k_stage item claims on their own L2 line (tailc[96])
#endif
#ifndef CC_STAGE_ECR
#define CC_STAGE_ECR 0       // 1: the refractory-gap fatigue decay staged with the factors
#endif
#ifndef CC_TAIL_STOP
#define CC_TAIL_STOP 10
#endif
#ifndef CC_BALANCED_ITEMS
#define CC_BALANCED_ITEMS 0  // k_plan: a group's work items of about equal size (measured: no gain)
#endif
#ifndef CC_REFR_BOOST
#define CC_REFR_BOOST 2      // queue classes a group with a refractory neuron moves up
#endif
#ifndef CC_CSR_STREAM
#define CC_CSR_STREAM 0
#endif
#ifndef CC_EVREC_STREAM
#define CC_EVREC_STREAM 0
#endif
#ifndef CC_TIMING_PROBES
#define CC_TIMING_PROBES 0   // timestamp / skip probes of the tools/*_timeline.py variants
#endif

namespace {


struct Ev {                              // one input event, 16 B
    double t;                            // arrival time, ms
    uint32_t src;                        // source gid (CC_EXT_SRC for the drive)
    float w;                             // recurrent weight (f32 as stored)
};

__device__ __forceinline__ long long pos_mod(long long a, long long m) {
    long long r = a % m;
    return r < 0 ? r + m : r;
}

// (t_mod + delta) mod L for |delta| <= L, given t_mod = t mod L: the log slot
// of step t + delta without a 64-bit modulo at every use.
__device__ __forceinline__ int slot_add(int t_mod, int delta, int L) {
    int e = t_mod + delta;
    if (e < 0) e += L;
    else if (e >= L) e -= L;
    return e;
}

// a / b, correctly rounded, for a constant divisor with rb = RN(1/b) (host
// float64): q0 = RN(a rb) is within 1 ulp of a/b, r = a - q0 b is exact in one
// FMA, and RN(q0 + r rb) = RN(a/b) (Markstein's theorem; no under/overflow for
// the time differences and tau constants here).  3 fp64 ops instead of the
// 14-instruction Newton division with its slow-path check.
__device__ __forceinline__ double div_rn(double a, double b, double rb) {
    const double q0 = __dmul_rn(a, rb);
    const double r = __fma_rn(-q0, b, a);
    return __fma_rn(r, rb, q0);
}

// Exponentials of the decay factors (np.exp / np.expm1 in _voltage_decay,
// model.py:131-138, and advance, model.py:280).  The reference's values come
// from numpy's SIMD routines, within 1 ulp of the exact result; any <= 1 ulp
// implementation reproduces its rasters.  These
// are shorter than libdevice's degree-11 polynomials on the hot path:
//   fexp    e^x = 2^(k/32) e^r, k = rint(32 x / ln2), |r| <= ln2/64; 2^(j/32) from
//           a table as hi + lo (the hi part correctly rounded), e^r - 1 by a
//           degree-6 Taylor polynomial (truncation < 0.03 ulp); 0.6 % of results
//           differ from the correctly rounded value by 1 ulp (np.exp: 5.6 %),
//           none by more (tools/micro/fexp.c, 1e7 arguments; tests/test_gpu_parity.py)
//   fexpm1  |x| <= 1/16: x + x^2 (1/2! + x/3! + ... + x^10/12!)
// Outside their ranges both fall back to libdevice.  The table lives in
// shared memory (k_stage copies it at entry).
__constant__ double2 c_exp2_tab[32] = {
    {0x1.0000000000000p+0, 0x0.0p+0}, {0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55},
    {0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54}, {0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54},
    {0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55}, {0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54},
    {0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54}, {0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55},
    {0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55}, {0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54},
    {0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55}, {0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59},
    {0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56}, {0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55},
    {0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54}, {0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54},
    {0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54}, {0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55},
    {0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55}, {0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54},
    {0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54}, {0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57},
    {0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56}, {0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54},
    {0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54}, {0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56},
    {0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55}, {0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56},
    {0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55}, {0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54},
    {0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54}, {0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54}};

__device__ __forceinline__ double fexp(double x, const double2* xt) {
    if (!(x > -700.0 && x < 700.0)) return exp(x);             // NaN / extreme: libdevice
    const double sh = 6755399441055744.0;                      // 1.5 * 2^52
    const double kd = __fma_rn(x, 0x1.71547652b82fep+5, sh);            // 32 / ln2
    const int k = __double2loint(kd);
    const double kf = __dsub_rn(kd, sh);
    double r = __fma_rn(kf, -0x1.62e42fefa39efp-6, x);                   // ln2/32 (hi)
    r = __fma_rn(kf, -0x1.abc9e3b39803fp-61, r);                          // ln2/32 (lo)
    double p = __fma_rn(r, 1.0 / 720.0, 1.0 / 120.0);
    p = __fma_rn(r, p, 1.0 / 24.0);
    p = __fma_rn(r, p, 1.0 / 6.0);
    p = __fma_rn(r, p, 0.5);
    p = __fma_rn(r, p, 1.0);
    p = __dmul_rn(p, r);                                       // e^r - 1
    const double2 t = xt[k & 31];
    const double y = __dadd_rn(t.x, __fma_rn(t.x, p, t.y));
    return __hiloint2double(__double2hiint(y) + ((k >> 5) << 20), __double2loint(y));
}

__device__ __forceinline__ double fexpm1(double x) {
    if (!(fabs(x) <= 0.0625)) return expm1(x);
    double p = __fma_rn(x, 1.0 / 479001600.0, 1.0 / 39916800.0);
    p = __fma_rn(x, p, 1.0 / 3628800.0);
    p = __fma_rn(x, p, 1.0 / 362880.0);
    p = __fma_rn(x, p, 1.0 / 40320.0);
    p = __fma_rn(x, p, 1.0 / 5040.0);
    p = __fma_rn(x, p, 1.0 / 720.0);
    p = __fma_rn(x, p, 1.0 / 120.0);
    p = __fma_rn(x, p, 1.0 / 24.0);
    p = __fma_rn(x, p, 1.0 / 6.0);
    p = __fma_rn(x, p, 0.5);
    return __fma_rn(__dmul_rn(x, x), p, x);
}

// Free evolution of one neuron to time te (NeuronBlock.advance,
// model.py:272-287 with _voltage_decay, model.py:116-143).
struct NState { double V, c, last, ru; };

__device__ __forceinline__ void advance(NState& s, const cc_pop& P, double te) {
    const double ff = fmin(fmax(s.last, s.ru), te);            // free_from
    double cs = s.c;
    if (ff != s.last && cs != 0.0)                             // exp(-0/tau) == 1 exactly
        cs = cs * exp(-div_rn(ff - s.last, P.tau_c, P.r_tau_c));
    const double Vs = (s.last < s.ru) ? P.V_r : s.V;
    const double dt = te - ff;
    // dt == 0: em = exp(-0/tau) = 1 and f = 0 * 1 exactly
    const double em = dt == 0.0 ? 1.0 : exp(-div_rn(dt, P.tau_m, P.r_tau_m));
    double Vt = P.E + (Vs - P.E) * em;
    double ct = cs;
    if (cs != 0.0 && dt != 0.0) {
        // with c == 0 the fatigue term is (sfa*0)*f == 0 for the always
        // finite f, and c*ec == 0: both skipped exactly
        const double ec = exp(-div_rn(dt, P.tau_c, P.r_tau_c));
        const double x = div_rn(dt * P.k1, P.k2, P.r_k2);
        double f;
        if (x == 0.0)
            f = dt * em;
        else if (fabs(x) <= 1.0)
            f = dt * em * expm1(x) / x;
        else
            f = dt * (ec - em) / x;
        Vt = Vt - P.sfa * cs * f;
        ct = cs * ec;
    } else if (cs != 0.0) {
        Vt = Vt - P.sfa * cs * 0.0;                            // f = dt * em = +0
    }
    s.V = (te < s.ru) ? P.V_r : Vt;
    s.c = ct;
    s.last = te;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t& total) {
    const int lane = threadIdx.x & 31;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

// A group's input lists: CC_SUBLISTS sub-lists (delivery of delay d appends to
// sub-list d % CC_SUBLISTS, spreading the reservation atomics over more
// counters), read as one concatenation.  init: lane j < CC_SUBLISTS holds the
// record count of sub-list j; every lane gets the exclusive prefix.
constexpr int NSUB = CC_SUBLISTS;
struct SubMap {
    uint32_t pre[NSUB + 1];
    __device__ __forceinline__ void init(uint32_t cj) {
        uint32_t x = 0;
#pragma unroll
        for (int j = 0; j < NSUB; ++j) { pre[j] = x; x += __shfl_sync(0xffffffffu, cj, j); }
        pre[NSUB] = x;
    }
    __device__ __forceinline__ uint32_t pre_at(int j) const {      // pre[j], j not a constant
        uint32_t v = pre[0];
#pragma unroll
        for (int i = 1; i <= NSUB; ++i)
            if (j >= i) v = pre[i];
        return v;
    }
    // record index of concatenated position r (< pre[NSUB]) in the group's region
    __device__ __forceinline__ size_t at(uint32_t r, size_t ks) const {
        int j = 0;
        uint32_t base = 0;
#pragma unroll
        for (int i = 1; i < NSUB; ++i)
            if (r >= pre[i]) { j = i; base = pre[i]; }
        return (size_t)j * ks + (r - base);
    }
};

// Append one spike to the log slot of emission step t: time, gid, row start
// and the row's delay-segment offsets (the delay-d part of its row is
// delivered in step t + d).  len == 0: no synapse on this shard.
// Returns the entry's reference (slot * spk_cap + index), CC_NO_REF if none.
constexpr uint32_t CC_NO_REF = 0xffffffffu;
__device__ __forceinline__ uint32_t log_spike(const cc_shard& sh, long long t, int e, uint32_t gid,
                                              double te) {
    CC_CHK(sh.ctl, gid < (uint32_t)sh.n_rows);
    const int64_t r0 = sh.row_off[gid];
    const int64_t len = sh.row_off[gid + 1] - r0;
    if (len == 0) return CC_NO_REF;
    const unsigned long long idx = atomicAdd(&sh.log_ctr[e], 1ull);
    if (idx >= (unsigned long long)sh.spk_cap) {
        cc_raise(sh.ctl, CC_ERR_SPIKE_LOG, t);
        return CC_NO_REF;
    }
    atomicAdd(&sh.log_len[e], (unsigned long long)len);
    const uint32_t ref = (uint32_t)(e * sh.spk_cap + idx);
    sh.log_t[ref] = te;
    sh.log_gid[ref] = gid;
    sh.log_r0[ref] = r0;
    const uint4* src = reinterpret_cast<const uint4*>(sh.dseg + (size_t)gid * sh.seg_stride);
    uint4* dst = reinterpret_cast<uint4*>(sh.log_dseg + (size_t)ref * sh.seg_stride);
    for (int j = 0; j < sh.seg_stride / 8; ++j) dst[j] = src[j];
    return ref;
}

// Warp-wide log_spike for received spikes (every lane calls; `valid` lanes
// carry a spike): one reservation atomic per warp instead of one per spike.
__device__ __forceinline__ void log_spike_warp(const cc_shard& sh, long long t, int e, bool valid,
                                               uint32_t gid, double te) {
    const int lane = threadIdx.x & 31;
    int64_t r0 = 0, len = 0;
    if (valid) {
        CC_CHK(sh.ctl, gid < (uint32_t)sh.n_rows);
        r0 = sh.row_off[gid];
        len = sh.row_off[gid + 1] - r0;
    }
    const bool has = valid && len > 0;
    const unsigned b = __ballot_sync(0xffffffffu, has);
    if (!b) return;
    unsigned long long lsum = has ? (unsigned long long)len : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    const int leader = __ffs(b) - 1;
    unsigned long long base = 0;
    if (lane == leader) {
        base = atomicAdd(&sh.log_ctr[e], (unsigned long long)__popc(b));
        atomicAdd(&sh.log_len[e], lsum);
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!has) return;
    const unsigned long long idx = base + (unsigned long long)__popc(b & ((1u << lane) - 1u));
    if (idx >= (unsigned long long)sh.spk_cap) {
        cc_raise(sh.ctl, CC_ERR_SPIKE_LOG, t);
        return;
    }
    const uint32_t ref = (uint32_t)(e * sh.spk_cap + idx);
    sh.log_t[ref] = te;
    sh.log_gid[ref] = gid;
    sh.log_r0[ref] = r0;
    const uint4* src = reinterpret_cast<const uint4*>(sh.dseg + (size_t)gid * sh.seg_stride);
    uint4* dst = reinterpret_cast<uint4*>(sh.log_dseg + (size_t)ref * sh.seg_stride);
    for (int j = 0; j < sh.seg_stride / 8; ++j) dst[j] = src[j];
}

// System-scope release / acquire of the peer exchange's flag words.
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Set by any thread of a k_stage block that pushed a spike to a peer this
// step: only those blocks need the system-scope fence before retiring.
__device__ __forceinline__ int& x_pushed_block() {
    __shared__ int flag;
    return flag;
}

// Peer exchange, send half: push one spike into the region of every
// destination rank in mask m (NVLink stores into the peer's window).
__device__ __forceinline__ void x_push(const cc_shard& sh, long long t, uint32_t m, uint32_t gid,
                                       double te) {
    const unsigned long long tb = (unsigned long long)__double_as_longlong(te);
    while (m) {
        const int d = __ffs(m) - 1;
        m &= m - 1;
        CC_CHK(sh.ctl, d < sh.n_ranks && sh.xdst[d].flag[0] != 0);
        const cc_xpeer& X = sh.xdst[d];
        x_pushed_block() = 1;
        const unsigned o = atomicAdd(&sh.xcnt[d], 1u);
        if (o < X.cap)
            reinterpret_cast<uint4*>(X.rec[t & 1])[o] =
                make_uint4(gid, (uint32_t)tb, (uint32_t)(tb >> 32), 0u);
        else
            cc_raise(sh.ctl, CC_ERR_XCAP, t);
    }
}

__device__ __forceinline__ Ev make_rec_event(const cc_shard& sh, uint64_t rec, int t_mod_l) {
    const uint32_t ref = (uint32_t)rec >> 5;                 // low 5 bits: lane in group
    CC_CHK(sh.ctl, ref < (uint32_t)(sh.log_slots * sh.spk_cap));
    const int e = (int)(ref >> (31 - __clz(sh.spk_cap)));      // spk_cap is a power of two
    CC_CHK(sh.ctl, (ref & (sh.spk_cap - 1)) < sh.log_ctr[e]);   // a logged entry
    int d = t_mod_l - e;
    if (d <= 0) d += sh.log_slots;
    Ev ev;
    // t_arr = t_emit + delay * dt (engine.py:364-365)
    ev.t = sh.log_t[ref] + (double)d * sh.dt;
    ev.src = sh.log_gid[ref];
    ev.w = __uint_as_float((uint32_t)(rec >> 32));
    return ev;
}

// ------------------------------------------------------------------ k_stage
// The neuron step.  One warp owns 32 consecutive neurons; their
// inputs pass through the warp's shared-memory buffer in rounds and every
// stage is spread over the 32 lanes:
//   1 gather   recurrent records (owner-major, 4 loads in flight per lane),
//              overflow surplus, external Poisson events
//   2 sort     per neuron: counting sort on a monotone time bucket
//              b(t) = clamp(floor((t - t0) * NB_L / dt)), NB_L ~ 2 inputs,
//              then the exact (t, src) rank of each input inside its bucket
//   3 factors  em = exp(-dt/tau_m), ec, f (model.py:116-143) of every input,
//              flattened, assuming the step-start refractory window and
//              fatigue flag: exactly the values the serial update computes
//   4 update   per lane, in order: affine update, jump, strict threshold,
//              reset, refractory discard, spike emission; after a spike the
//              neuron's remaining factors are recomputed in line.
// Staging constants; overridable with -D for parameter sweeps (build(defines=...)).
// A sweep at config 1 (w 128..384, 4..16 fixed buckets, warps 2..4) put all variants
// within 12% of each other, the default among the best.
#ifndef CC_NEURON_WCAP
#define CC_NEURON_WCAP 256
#endif
#ifndef CC_STAGE_WARPS
#define CC_STAGE_WARPS 4
#endif
constexpr int NEURON_WCAP = CC_NEURON_WCAP;   // events per round (8 per lane)
constexpr int STAGE_WARPS = CC_STAGE_WARPS;

// Sort buckets per work item: neuron L gets NB_L = min(2 n_L, 352 n_L / rtot + 1)
// buckets (0 if it has no input), so sum NB_L <= HCAP and a bucket holds ~0.5
// inputs on average.
#ifndef CC_HCAP
#define CC_HCAP 280
#endif
constexpr int HCAP = CC_HCAP;

struct StageBuf {
    double* t; double* o_last; double* o_ru; double* bsc;
    uint32_t* src; float* w; uint32_t* keep; uint32_t* hist; int* seg; uint32_t* o_flag;
    uint32_t* cbk;
    uint16_t* perm; uint16_t* prov; uint8_t* own; uint8_t* owns;
};

__host__ __device__ constexpr size_t stage_warp_bytes() {
    return ((size_t)NEURON_WCAP * (8 + 4 + 4 + 4 + 2 + 2 + 1 + 1) + HCAP * 4 + 34 * 4
            + 32 * (8 + 8 + 8 + 4 + 4) + 32 + 15) / 16 * 16;     // 16 B aligned per warp
}

// dynamic shared memory of k_stage behind the warps' buffers: the tail
// delivery's unit tables a_n[d_max], a_pre[d_max + 1]
static inline size_t stage_tail_bytes(int d_max) {
    return ((size_t)(2 * d_max + 1) * 4 + 15) / 16 * 16;
}

__device__ __forceinline__ StageBuf carve(char* p) {
    StageBuf b;
    b.t = (double*)p; p += NEURON_WCAP * 8;
    b.o_last = (double*)p; p += 32 * 8;
    b.o_ru = (double*)p; p += 32 * 8;
    b.bsc = (double*)p; p += 32 * 8;
    b.src = (uint32_t*)p; p += NEURON_WCAP * 4;
    b.w = (float*)p; p += NEURON_WCAP * 4;
    b.keep = (uint32_t*)p; p += NEURON_WCAP * 4;
    b.hist = (uint32_t*)p; p += HCAP * 4;
    b.seg = (int*)p; p += 34 * 4;
    b.o_flag = (uint32_t*)p; p += 32 * 4;
    b.cbk = (uint32_t*)p; p += 32 * 4;
    b.perm = (uint16_t*)p; p += NEURON_WCAP * 2;
    b.prov = (uint16_t*)p; p += NEURON_WCAP * 2;
    b.own = (uint8_t*)p; p += NEURON_WCAP;
    b.owns = (uint8_t*)p;
    return b;
}

// decay factors of one event (the dt-dependent part of _voltage_decay)
__device__ __forceinline__ void decay_factors(const cc_pop& P, double dt, bool with_c,
                                              double& em, double& ec, double& f,
                                              const double2* xt) {
    ec = 1.0;
    f = 0.0;
    if (dt == 0.0) {            // exp(-0/tau) == 1, x == 0 -> f = 0 * 1: exact shortcut
        em = 1.0;
        return;
    }
    em = fexp(-div_rn(dt, P.tau_m, P.r_tau_m), xt);
    if (with_c) {
        ec = fexp(-div_rn(dt, P.tau_c, P.r_tau_c), xt);
        const double x = div_rn(dt * P.k1, P.k2, P.r_k2);
        if (x == 0.0)
            f = dt * em;
        else if (fabs(x) <= 1.0)
            f = dt * em * fexpm1(x) / x;
        else
            f = dt * (ec - em) / x;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}


// Timing probes (tools/*_timeline.py; compiled only with -DCC_TIMING_PROBES=1):
// flags & 32: per work item of k_stage, 8 timestamps
// {claim, gathered, sorted, factors, updated, update start (0: none), rtot, warp} written to the
// tail of the scratch buffer.
#define CC_DBG(slot_i, val)                                                              \
    do {                                                                                 \
        if (CC_TIMING_PROBES && (sh.flags & 32) && lane == 0 && item < 65536u) {          \
            unsigned long long* d_ = reinterpret_cast<unsigned long long*>(sh.scratch)    \
                                     + (size_t)sh.scratch_cap * 7 - (size_t)(item + 1) * 8; \
            d_[slot_i] = (val);                                                          \
        }                                                                                \
    } while (0)

__device__ __forceinline__ int neuron_pop(const cc_shard& sh, uint32_t gid) {
    return ((int)(gid % (uint32_t)sh.n_col) < sh.n_exc_col) ? 0 : 1;
}

// General (rare) step of the in-order update: refractory window involved or
// factors invalidated by an earlier spike in this step.  Returns true when the
// strict threshold is crossed.  ecr0 = exp(-(ff - last) / tau_c) as staged
// (valid unless stale, like em0, ec0, f0).
__device__ __forceinline__ bool slow_step(NState& s, const cc_pop& P, double tj, bool stale,
                                       bool cflag, double em0, double ec0, double f0,
                                       double ecr0, double w, const double2* xt) {
    const double ff = fmin(fmax(s.last, s.ru), tj);
    double cs = s.c;
    if (ff != s.last && cs != 0.0) {                  // leaving / inside a refractory window
#if CC_STAGE_ECR
        if (stale) cs = cs * fexp(-div_rn(ff - s.last, P.tau_c, P.r_tau_c), xt);
        else cs = cs * ecr0;
#else
        cs = cs * fexp(-div_rn(ff - s.last, P.tau_c, P.r_tau_c), xt);
#endif
    }
    double emj = em0, ecj = ec0, fj = f0;
    if (stale) decay_factors(P, tj - ff, cs != 0.0, emj, ecj, fj, xt);
    else if (!cflag) { ecj = 1.0; fj = 0.0; }
    // model.py:116-143 and 272-287, reference op order
    const double Vs = (s.last < s.ru) ? P.V_r : s.V;
    double Vt = P.E + (Vs - P.E) * emj;
    double ct = cs;
    if (cs != 0.0) {
        Vt = Vt - P.sfa * cs * fj;
        ct = cs * ecj;
    }
    s.V = (tj < s.ru) ? P.V_r : Vt;
    s.c = ct;
    s.last = tj;
    if (tj >= s.ru) {
        const double V = s.V + w;
        if (V > P.V_theta) return true;
        s.V = V;
    } else {
        s.V = P.V_r;                                  // refractory: input discarded
    }
    return false;
}

// ------------------------------------------------------------ delivery
// A work unit is (delay d, 4 consecutive spikes of log slot t - d); each spike's
// delay-d segment is walked by 8 lanes, U synapses per lane per pass.  Records
// are deposited into the per-group input lists of the arrival step.
#ifndef CC_DEL_THREADS
#define CC_DEL_THREADS 256
#endif
#ifndef CC_DEL_MINB
#define CC_DEL_MINB 2
#endif
#ifndef CC_DEL_U
#define CC_DEL_U 8          // synapses per lane per pass
#endif
// Lanes per spike: 8 (4 spikes per unit) or 16 (2 per unit), chosen per shard
// by the host (sh.del_lps_log2); the k_stage tail and k_deliver share it.
__device__ __forceinline__ int del_lps(const cc_shard& sh) { return 1 << sh.del_lps_log2; }
constexpr int DEL_DMAX = 256;               // d_max <= 255 (uint8 delays)

// Input lists of arrival step t: two sets (t & 1), so that step t+1's
// delay >= 2 events can be delivered while step t is integrated.
struct ListSet { uint32_t* cnt; uint64_t* rec; uint32_t* ovf_cnt; uint4* ovf; };
__device__ __forceinline__ ListSet list_set(const cc_shard& sh, long long t) {
    const int s = (int)(t & 1);
    ListSet S;
    S.cnt = sh.bin_cnt + (size_t)s * sh.n_groups * NSUB * CC_CNT_STRIDE;
    S.rec = sh.bin_rec + (size_t)s * sh.n_groups * NSUB * ((size_t)sh.bin_cap + sh.bin_pad);
    S.ovf_cnt = sh.ovf_cnt + s;
    S.ovf = reinterpret_cast<uint4*>(sh.ovf_rec) + (size_t)s * sh.ovf_cap;
    return S;
}

// Unit space of an arrival step: position k = 0..D-1 holds delay d = k + 2 for
// k < D - 1 and d = 1 for k = D - 1 - the delay >= 2 units first, since their
// spikes are all logged a step ahead.
__device__ __forceinline__ int unit_delay(int k, int D) { return k < D - 1 ? k + 2 : 1; }

// Block-wide (barriers): s_n[k] spikes of log slot ta - d(k), s_pre the unit
// prefix over positions k < nk.
__device__ __forceinline__ void unit_prefix(const cc_shard& sh, int ta_mod, int nk,
                                            unsigned* s_n, unsigned* s_pre) {
    if (threadIdx.x < 32) {                  // warp 0: loads and a shuffle scan, 32 at a time
        const int lane = threadIdx.x;
        unsigned carry = 0;
        for (int k0 = 0; k0 < nk; k0 += 32) {
            const int k = k0 + lane;
            unsigned n = 0;
            if (k < nk)
                n = (unsigned)min(sh.log_ctr[slot_add(ta_mod, -unit_delay(k, sh.d_max),
                                                      sh.log_slots)],
                                  (unsigned long long)sh.spk_cap);
            const unsigned units = (n + (32u >> sh.del_lps_log2) - 1) >> (5 - sh.del_lps_log2);
            unsigned tot;
            const unsigned ex = warp_excl_scan(units, tot);
            if (k < nk) { s_n[k] = n; s_pre[k] = carry + ex; }
            carry += tot;
        }
        if (lane == 0) s_pre[nk] = carry;
    }
    __syncthreads();
}

// This lane's spike of unit u (< s_pre[nk]) of arrival step ta: segment start,
// length and log reference; kc is the caller's position cursor (its units
// only increase).
__device__ __forceinline__ void unit_desc(const cc_shard& sh, int ta_mod, const unsigned* s_n,
                                          const unsigned* s_pre, unsigned u, int& kc,
                                          uint64_t& st, uint32_t& ln, uint32_t& rf) {
    while (s_pre[kc + 1] <= u) ++kc;
    const unsigned idx = ((u - s_pre[kc]) << (5 - sh.del_lps_log2)) + ((threadIdx.x & 31) >> sh.del_lps_log2);
    st = 0; ln = 0; rf = 0;
    if (idx < s_n[kc]) {
        const int d = unit_delay(kc, sh.d_max);
        CC_CHK(sh.ctl, d >= 1 && d <= sh.d_max && idx < (unsigned)sh.spk_cap);
        const int e = slot_add(ta_mod, -d, sh.log_slots);
        rf = (uint32_t)(e * sh.spk_cap + idx);
        const uint16_t* ds = sh.log_dseg + (size_t)rf * sh.seg_stride;
        const uint32_t a = __ldg(ds + d - 1), b = __ldg(ds + d);
        st = (uint64_t)__ldg(sh.log_r0 + rf) + a;
        ln = b - a;
    }
}

__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int U>
__device__ __forceinline__ void load_pass(const cc_shard& sh, uint64_t st, uint32_t ln, int p,
                                          int* tg, float* w) {
    const int lps = del_lps(sh);
    const int sl = threadIdx.x & (lps - 1);
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t j = (uint32_t)((p * U + u) * lps + sl);
        tg[u] = -1;
        if (j < ln) {
            CC_CHK(sh.ctl, st + j < (uint64_t)sh.row_off[sh.n_rows]);
            tg[u] = __ldg(sh.syn_tgt + st + j);
            w[u] = __ldg(sh.syn_w + st + j);
            CC_CHK(sh.ctl, tg[u] >= 0 && tg[u] < sh.n_local);
        }
    }
}

// Reserve and deposit one pass: one atomic per run of consecutive lanes with
// the same group (a segment is sorted by target, network.py:257, so a spike's
// 8 lanes form 1-3 runs; runs are found with a shuffle and a ballot); lists
// that are full spill to the set's overflow list.
#ifndef CC_SUB_BY_LANE
#define CC_SUB_BY_LANE 1     // sub-lists by target lane range (0: by delay, `sub` of the caller)
#endif
static_assert((NSUB & (NSUB - 1)) == 0 && NSUB <= 32, "CC_SUBLISTS must be a power of two <= 32");
__device__ __forceinline__ unsigned list_of(int tg, int sub) {
#if CC_SUB_BY_LANE
    return ((unsigned)tg * NSUB) >> 5;                  // (tg >> 5) * NSUB + (tg & 31) * NSUB / 32
#else
    return ((unsigned)tg >> 5) * NSUB + (unsigned)sub;
#endif
}

template <int U>
__device__ __forceinline__ void deposit_pass(const cc_shard& sh, const ListSet& S, int sub,
                                             const int* tg, const float* w, uint32_t rf,
                                             long long t_err) {
    const int lane = threadIdx.x & 31;
    const int K = sh.bin_cap;
    const size_t KS = (size_t)K + sh.bin_pad;
    unsigned key[U], pos[U], got[U];
    int lead[U];
    const unsigned upto = 0xffffffffu >> (31 - lane);      // bits 0..lane
#pragma unroll
    for (int k = 0; k < U; ++k) {
        // list of the target: group * NSUB + sub-list; with CC_SUB_BY_LANE the
        // sub-list is the target's lane range (NSUB ranges of 32 / NSUB lanes)
        key[k] = tg[k] >= 0 ? list_of(tg[k], sub) : 0xffffffffu;
        CC_CHK(sh.ctl, tg[k] < 0 || key[k] < (unsigned)sh.n_groups * NSUB);
        const unsigned prev = __shfl_up_sync(0xffffffffu, key[k], 1);
        const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || key[k] != prev);
        lead[k] = 31 - __clz(heads & upto);
        const unsigned after = heads & ~upto;
        const int end = after ? __ffs(after) - 1 : 32;
        got[k] = 0u;
        if (tg[k] >= 0 && lane == lead[k]) {
            if (CC_TIMING_PROBES && (sh.flags & 1024)) got[k] = 0u;   // probe: no reservation
            else got[k] = atomicAdd(&S.cnt[(size_t)key[k] * CC_CNT_STRIDE],
                                    (unsigned)(end - lead[k]));
        }
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
        pos[k] = __shfl_sync(0xffffffffu, got[k], lead[k]) + (unsigned)(lane - lead[k]);
#pragma unroll
    for (int k = 0; k < U; ++k) {
        if (tg[k] < 0 || (CC_TIMING_PROBES && (sh.flags & 2048))) continue;  // probe: no deposit
        const uint32_t lig = (uint32_t)tg[k] & 31u;
        if (pos[k] < (unsigned)K) {
            S.rec[(size_t)key[k] * KS + pos[k]] =
                (uint64_t)((rf << 5) | lig) | ((uint64_t)__float_as_uint(w[k]) << 32);
        } else {
            const unsigned o = atomicAdd(S.ovf_cnt, 1u);
            atomicAdd(&sh.ctl->ovf_total, 1ull);
            if (o < (unsigned)sh.ovf_cap)
                S.ovf[o] = make_uint4((unsigned)tg[k] >> 5, lig, rf, __float_as_uint(w[k]));
            else cc_raise(sh.ctl, CC_ERR_OVERFLOW_BIN, t_err);
        }
    }
}

// Planning pass of phase A: per group of 32 neurons, the input counts
// (ring-slot occupancy and the Poisson draw), the group's stream region and
// its split into work items ("rounds") of at most NEURON_WCAP inputs, appended
// to a global queue so that heavy groups are spread over many warps.
// Block-wide (barriers): every warp of the block plans group group0 (or idles
// if group0 is past the last group).
__device__ __forceinline__ void plan_group(const cc_shard& sh, long long t, int group0) {
    const unsigned long long pt0 = gtimer();
    cc_ctl* ctl = sh.ctl;
    // (after a failed run the plan is still bounded - every write is checked -
    // and k_stage processes nothing; the block barriers below need all warps)
    const int lane = threadIdx.x & 31;
    const bool gvalid = group0 * 32 < sh.n_local;   // warps past the last group idle
    const int group = gvalid ? group0 : 0;
    const int li = group * 32 + lane;
    const bool active = gvalid && li < sh.n_local;
    // inputs of this step: count the group's list records per lane
    __shared__ uint32_t lane_cnt[8][32];
    const int wib = threadIdx.x >> 5;
    lane_cnt[wib][lane] = 0u;
    const uint32_t K = (uint32_t)sh.bin_cap;
    const size_t KS = (size_t)K + sh.bin_pad;
    const ListSet S = list_set(sh, t);
    uint32_t* gcb = S.cnt + (size_t)group * NSUB * CC_CNT_STRIDE;
    const uint32_t cj_all = (gvalid && lane < NSUB) ? gcb[lane * CC_CNT_STRIDE] : 0u;
    const uint32_t cj = min(cj_all, K);
    SubMap M;
    M.init(cj);
    const uint32_t c_list = M.pre[NSUB];
    uint32_t ovf_all = cj_all - cj;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ovf_all += __shfl_xor_sync(0xffffffffu, ovf_all, o);
    const long long o0 = sh.ovf_off[group];
    const uint32_t c_ovf = ovf_all ? (uint32_t)max(0ll, min((long long)ovf_all, sh.ovf_cap - o0)) : 0u;
    __syncwarp();
    const uint64_t* lst = S.rec + (size_t)group * NSUB * KS;
    // routed delivery with per-neuron counts: k_bin counted the records it
    // stored per neuron (every list record of the step came through it), so the
    // records need not be read here; the counts are zeroed for step t + 2
    if (sh.l1_ncnt) {
        if (gvalid) {
            uint32_t* nc = sh.l1_ncnt + (size_t)(t & 1) * sh.n_groups * 32 + (size_t)group * 32 + lane;
            lane_cnt[wib][lane] = *nc;
            *nc = 0u;
        }
        __syncwarp();
    }
    for (uint32_t r0 = 0; r0 < (sh.l1_ncnt ? 0u : c_list); r0 += 32 * 8) {
        uint32_t v[8];                             // 8 loads in flight per lane
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t r = r0 + u * 32 + lane;
            v[u] = r < c_list ? (uint32_t)lst[M.at(r, KS)] : 0xffffffffu;   // ref < 2^27: never all-ones
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (v[u] != 0xffffffffu) atomicAdd(&lane_cnt[wib][v[u] & 31u], 1u);
    }
    const uint4* ov = reinterpret_cast<const uint4*>(sh.ovf_sorted) + o0;
    // (& 31: after an overflow-list error the slots of dropped records hold
    // stale data; the run is failed then, but shared memory stays in bounds)
    for (uint32_t r = lane; r < c_ovf; r += 32) atomicAdd(&lane_cnt[wib][ov[r].y & 31u], 1u);
    __syncwarp();
    if (gvalid && lane < NSUB) {
        gcb[lane * CC_CNT_STRIDE] = 0u;            // drain the lists (read back via grp_sub)
        sh.grp_sub[(size_t)group * NSUB + lane] = cj;
    }
    if (lane == 0 && gvalid) sh.grp_n[group] = c_list + c_ovf;
    const unsigned long long pt1 = gtimer();
    uint32_t n_r = 0, n_e = 0;
    if (active) {
        const uint32_t gid = sh.gid[li];
        n_r = lane_cnt[wib][lane];
        if (sh.ext_budget > 0) {
            // Poisson count by product of uniforms (engine.py:172-188): the
            // prefix product never increases, so stopping at the first
            // product <= exp(-lambda) counts exactly the same terms.
            const uint64_t h4 = cc_splitmix64(cc_splitmix64(sh.h2_ext ^ (uint64_t)gid)
                                              ^ (uint64_t)t);
            // uniforms 4 at a time (independent hashes), products in order
            double prod = 1.0;
            int k = sh.ext_budget;
            for (int k0 = 0; k0 < sh.ext_budget; k0 += 4) {
                double u[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) u[j] = cc_u53(cc_splitmix64(h4 ^ (uint64_t)(k0 + j)));
                bool done = false;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (done || k0 + j >= sh.ext_budget) continue;
                    prod = prod * u[j];
                    if (!(prod > sh.ext_thresh)) { k = k0 + j; done = true; }
                }
                if (done) break;
            }
            if (k >= sh.ext_budget) cc_raise(ctl, CC_ERR_POISSON, t);
            n_e = (uint32_t)k;
        }
    }
    const uint32_t n = n_r + n_e;
    const unsigned long long pt2 = gtimer();
    uint32_t nmax = n;
    unsigned long long es = n_e;
    uint32_t mb = n_r;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
        es += __shfl_xor_sync(0xffffffffu, es, o);
    }
    if (active) {
        sh.ev_n[li] = (int32_t)n;
        sh.ev_nr[li] = (int32_t)n_r;
    }
    // greedy split of lanes 0..31 into items of <= NEURON_WCAP inputs (a lane
    // with more forms an item alone), warp-parallel: lane s finds by binary
    // search the first lane e > s whose inclusive prefix exceeds
    // prefix(s - 1) + NEURON_WCAP; the items are the chain first, e(first), ...
    // Items are queued by the size class of their group, heaviest first, so
    // that the last items claimed (and group updates run) are short.
    const uint32_t nn = active ? n : 0u;
    uint32_t gtot;
    const uint32_t excl = warp_excl_scan(nn, gtot);
    const uint32_t incl = excl + nn;
    // item size limit: NEURON_WCAP, or (CC_BALANCED_ITEMS) the group's total
    // split evenly over the fewest items that hold it, plus one neuron's worth
    // of slack so that whole lanes still pack into that many items - a 415-input
    // group becomes ~230 + ~185 instead of ~250 + ~165, and the longest item of
    // a round of items (which every warp of the round waits behind) is shorter
    uint32_t icap = (uint32_t)NEURON_WCAP;
    if (CC_BALANCED_ITEMS && gtot > (uint32_t)NEURON_WCAP) {
        const uint32_t k = (gtot + NEURON_WCAP - 1) / NEURON_WCAP;
        icap = min(icap, (gtot + k - 1) / k + nmax);
    }
    const uint32_t thr = excl + icap;
    int lo = lane + 1, hi = 32;
#pragma unroll
    for (int it = 0; it < 6; ++it) {
        const int mid = (lo + hi) >> 1;
        const uint32_t pm = __shfl_sync(0xffffffffu, incl, mid & 31);
        if (lo < hi) {
            if (pm > thr) hi = mid; else lo = mid + 1;
        }
    }
    const unsigned has = __ballot_sync(0xffffffffu, nn > 0);
    int ni = 0;
    uint32_t my_item = 0;
    for (int st = has ? __ffs(has) - 1 : 32; st < 32; ++ni) {
        const int en = __shfl_sync(0xffffffffu, lo, st);
        if (lane == ni) my_item = (uint32_t)st | ((uint32_t)en << 8);
        st = en;
    }
    const unsigned long long pt3 = gtimer();
    if (lane == 0 && gvalid) sh.grp_items[group] = (uint32_t)ni;
    // queue positions: per-block counts per class, one global atomic per class
    __shared__ unsigned blk_cls[CC_ITEM_CLASSES], blk_base[CC_ITEM_CLASSES];
    __shared__ unsigned long long blk_es;
    __shared__ unsigned blk_ni, blk_mb, blk_nmax;
    if (threadIdx.x < CC_ITEM_CLASSES) blk_cls[threadIdx.x] = 0u;
    if (threadIdx.x == 0) { blk_es = 0ull; blk_ni = 0u; blk_mb = 0u; blk_nmax = 0u; }
    __syncthreads();
    int cls = 0;
    unsigned local = 0;
    // a neuron inside its refractory window at the step start takes the slow
    // step of the update for every input before the window ends (measured at
    // config 1: +0.38 us per slow step on a 9 us group update; the last groups
    // to finish were those of second-round items with 15-25 slow steps):
    // such groups move CC_REFR_BOOST classes up, so their updates start early
    bool boost = false;
    if (CC_REFR_BOOST > 0) {
        const bool refr = active && nn > 0 &&
                          sh.state[(size_t)li * 4 + 3] > (double)t * sh.dt;
        boost = __any_sync(0xffffffffu, refr);
    }
    if (lane < ni) {
        // class by the GROUP's input total: all items of a heavy group are
        // claimed early, so its (long) in-order update does not start last
        cls = CC_ITEM_CLASSES - 1 - (int)min(gtot / (uint32_t)NEURON_WCAP,
                                             (uint32_t)(CC_ITEM_CLASSES - 1));
        if (boost) cls = max(cls - CC_REFR_BOOST, 0);
        local = atomicAdd(&blk_cls[cls], 1u);
    }
    if (lane == 0) {
        if (ni) atomicAdd(&blk_ni, (unsigned)ni);
        if (es) atomicAdd(&blk_es, es);
        if (mb) atomicMax(&blk_mb, mb);
        if (nmax) atomicMax(&blk_nmax, nmax);
    }
    __syncthreads();
    if (threadIdx.x < CC_ITEM_CLASSES && blk_cls[threadIdx.x])
        blk_base[threadIdx.x] = atomicAdd(&ctl->cls_n[threadIdx.x], blk_cls[threadIdx.x]);
    if (threadIdx.x == 0) {
        if (blk_ni) atomicAdd(&ctl->n_rounds, blk_ni);
        if (blk_es) atomicAdd(&ctl->ext_events, blk_es);
        if (blk_mb) atomicMax(&ctl->max_bin, blk_mb);
        if (blk_nmax) atomicMax(&ctl->max_events, blk_nmax);
    }
    __syncthreads();
    if (lane < ni) {
        const unsigned at = blk_base[cls] + local;
        if (at >= (unsigned)sh.round_cap) {
            cc_raise(ctl, CC_ERR_SCRATCH, t);
        } else {
            uint32_t* r = sh.rounds + 2 * ((size_t)cls * sh.round_cap + at);
            r[0] = (uint32_t)group;
            r[1] = my_item;
        }
    }
    if (CC_TIMING_PROBES && (sh.flags & 512) && lane == 0 && gvalid) {
        unsigned long long* d_ = reinterpret_cast<unsigned long long*>(sh.scratch)
                                 + (size_t)sh.scratch_cap * 7 - (size_t)(group + 1) * 8;
        unsigned smid_;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid_));
        d_[0] = pt0; d_[1] = pt1; d_[2] = pt2; d_[3] = pt3; d_[4] = gtimer();
        d_[5] = smid_; d_[6] = c_list + c_ovf; d_[7] = (unsigned long long)ni;
    }
    __syncthreads();                               // block arrays reused by the next call
}

__global__ void __launch_bounds__(128)
k_plan(const cc_shard sh) {
    const long long t = *(volatile long long*)&sh.ctl->t;
    plan_group(sh, t, (blockIdx.x * blockDim.x + threadIdx.x) >> 5);
}

// Peer exchange: publish step t's per-destination record counts (last block
// of k_stage; every other block's pushes are ordered before by its system
// fence and the completion counter).  Every linked destination gets a flag
// every step, also with no records, so that all ranks advance in lockstep
// and a region is never rewritten before its receiver consumed it (the
// regions alternate by step parity).  Runs also after a device error (with
// the counts as they stand) so that peers never wait in vain.
__device__ __noinline__ void x_publish(const cc_xpeer* xdst, uint32_t* xcnt, int n_ranks,
                                      cc_ctl* ctl, long long t) {
    __threadfence_system();
    unsigned long long sent = 0;
    for (int d = 0; d < n_ranks; ++d) {
        const cc_xpeer& X = xdst[d];
        if (!X.flag[0]) continue;
        const uint32_t c = min(*(volatile uint32_t*)&xcnt[d], X.cap);
        xcnt[d] = 0u;
        sent += c;
        st_release_sys(reinterpret_cast<unsigned long long*>(X.flag[t & 1]),
                       ((unsigned long long)(t + 1) << 32) | c);
    }
    if (sent) ctl->x_sent += sent;
}

// In-order update of the 32 neurons of one group (NeuronBlock.integrate_sorted,
// model.py:289-337), one lane per neuron: affine update, jump, strict
// threshold, reset, refractory discard, spike emission.  The factors assume the
// step-start refractory window; after a spike they are recomputed in line
// (slow_step).  The ordered 48 B records {t, w}, {em, ec}, {f, ecr} reach the
// warp's (idle) shared buffer by cp.async (L2 only): CC_UPD_NBUF batches of
// one input per neuron each are in flight while one is applied, so a
// neuron's serial chain does not wait for an L2 round trip per input (1 input
// x 3 buffers: 97.2 -> 94.3 us per step at config 1; the single-buffer
// fallback, 5 inputs per round trip, serves builds whose buffer is too small).
constexpr int UB = stage_warp_bytes() / (32 * 48) < 5 ? (int)(stage_warp_bytes() / (32 * 48))
                                                        : 5;    // inputs per neuron per batch
constexpr int UB_STRIDE = 3 * UB;        // double2 per lane: 15 = 7 mod 8, conflict-free
static_assert(32 * UB_STRIDE * 16 <= stage_warp_bytes(), "update batch > stage buffer");
#ifndef CC_UPD_PIPE
#define CC_UPD_PIPE 1        // update: CC_UPD_NBUF single-input batches in flight
#endif
#ifndef CC_UPD_NBUF
#define CC_UPD_NBUF 3
#endif
static_assert(!CC_UPD_PIPE || CC_UPD_NBUF * 32 * 3 * 16 <= (int)stage_warp_bytes(),
              "update pipeline > stage buffer");

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

__device__ __forceinline__ void update_group(const cc_shard& sh, int li0, long long t, int e_t,
                                             double2* S, uint32_t& my_spikes,
                                             const double2* xt,
                                             [[maybe_unused]] unsigned long long* dbg_info = nullptr) {
    [[maybe_unused]] unsigned dbg_slow = 0, dbg_spk = 0;
    cc_ctl* ctl = sh.ctl;
    const int lane = threadIdx.x & 31;
    const int li = li0 + lane;
    const uint32_t n = li < sh.n_local ? (uint32_t)sh.ev_n[li] : 0u;
    const uint32_t off = n ? (uint32_t)__ldcg(&sh.ev_off[li]) : 0u;
    CC_CHK(sh.ctl, (unsigned long long)off + n <= (unsigned long long)sh.evrec_cap);
    uint32_t nmax = n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    const double2* R = reinterpret_cast<const double2*>(sh.evrec);
    uint32_t gid = 0;
    const cc_pop* P = &sh.pop[0];
    double* st = sh.state + (size_t)(n ? li : 0) * 4;
    NState s{0.0, 0.0, 0.0, 0.0};
    if (n) {
        gid = sh.gid[li];
        P = &sh.pop[neuron_pop(sh, gid)];
        const double2 a0 = reinterpret_cast<const double2*>(st)[0];
        const double2 a1 = reinterpret_cast<const double2*>(st)[1];
        s = NState{a0.x, a0.y, a1.x, a1.y};
    }
    const bool cflag = s.c != 0.0;
    bool stale = false;                      // spiked: factors need recomputing
#if CC_UPD_PIPE
    // CC_UPD_NBUF single-input buffers per lane in flight: input i+NBUF is
    // loading while input i is applied (cp.async groups, wait_group NBUF-1);
    // rotating buffer indices, one 48 B slot per lane and buffer
    double2* const sb = S + lane * 3;
    constexpr int BS = 32 * 3;                   // double2 per buffer
    const double2* Rp = R + 3 * (size_t)off;     // next record of this lane to fetch
    uint32_t jn = 0;                             // its input index
    int bn = 0, bi = 0;                          // buffer to fill next / to apply
    auto issue = [&]() {
        if (jn < n) {
            double2* d = sb + bn * BS;
            cp_async16(d, Rp);
            cp_async16(d + 1, Rp + 1);
            cp_async16(d + 2, Rp + 2);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        Rp += 3;
        ++jn;
        bn = bn + 1 == CC_UPD_NBUF ? 0 : bn + 1;
    };
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CC_UPD_NBUF; ++j) issue();
    // (each lane copies into and reads only its own slots, and cp.async waits
    // are per thread: no warp barrier inside the loop)
    for (uint32_t b0 = 0; b0 < nmax; ++b0) {
        asm volatile("cp.async.wait_group %0;" ::"n"(CC_UPD_NBUF - 1) : "memory");
        const double2* my = sb + bi * BS;
        bi = bi + 1 == CC_UPD_NBUF ? 0 : bi + 1;
        const uint32_t e = min(n, b0 + 1u);
#else
    const double2* my = S + lane * UB_STRIDE;
    for (uint32_t b0 = 0; b0 < nmax; b0 += UB) {
        __syncwarp();                        // previous batch consumed
        {
            const double2* Rn = R + 3 * (size_t)(off + b0);
            const uint32_t m = n > b0 ? min(n - b0, (uint32_t)UB) : 0u;
#pragma unroll
            for (int k = 0; k < UB; ++k) {
                if ((uint32_t)k < m) {
                    cp_async16(S + lane * UB_STRIDE + 3 * k, Rn + 3 * k);
                    cp_async16(S + lane * UB_STRIDE + 3 * k + 1, Rn + 3 * k + 1);
                    cp_async16(S + lane * UB_STRIDE + 3 * k + 2, Rn + 3 * k + 2);
                }
            }
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        const uint32_t e = min(n, b0 + (uint32_t)UB);
#endif
        for (uint32_t i = b0; i < e; ++i) {
            const double2 r0 = my[3 * (i - b0)], r1 = my[3 * (i - b0) + 1],
                          r2 = my[3 * (i - b0) + 2];
            const double tj = r0.x, wv = r0.y, em = r1.x, ec = r1.y, f = r2.x, ecr = r2.y;
            bool spike = false;
            if (!stale && s.ru <= s.last) {
                // fast path (no refractory window involved, factors valid):
                // free_from == last, V_s == V, not refractory; ec = 1, f = 0 when
                // the neuron started the step without fatigue (c stays 0 then)
                double Vt = P->E + (s.V - P->E) * em;
                if (s.c != 0.0) {
                    Vt = Vt - P->sfa * s.c * f;
                    s.c = s.c * ec;
                }
                s.last = tj;
                const double V = Vt + wv;
                if (V > P->V_theta) spike = true; else s.V = V;
            } else {
                if (CC_TIMING_PROBES) ++dbg_slow;
                spike = slow_step(s, *P, tj, stale, cflag, em, ec, f, ecr, wv, xt);
            }
            if (CC_TIMING_PROBES && spike) ++dbg_spk;
            if (spike) {                             // strict threshold crossed
                s.V = P->V_r;
                s.c = s.c + P->alpha_c;
                s.ru = tj + P->tau_arp;
                stale = true;
                ++my_spikes;
                if (sh.direct_log) log_spike(sh, t, e_t, gid, tj);
                if (sh.xdst) {                               // peer exchange: push now
                    const uint32_t xm = sh.xmask[li];
                    if (xm) x_push(sh, t, xm, gid, tj);
                }
                if ((!sh.direct_log && !sh.xdst) || (sh.remote && sh.remote[li])) {   // out-list
                    const unsigned o = atomicAdd(&ctl->out_n, 1u);
                    if (o < (unsigned)sh.out_cap) { sh.out_gid[o] = gid; sh.out_t[o] = tj; }
                    else cc_raise(ctl, CC_ERR_OUTLIST, t);
                }
                const unsigned long long rr = atomicAdd(&ctl->raster_n, 1ull);
                if (rr < (unsigned long long)sh.raster_cap) {
                    sh.raster_gid[rr] = gid;
                    sh.raster_t[rr] = tj;
                } else {
                    cc_raise(ctl, CC_ERR_RASTER, t);
                }
            }
        }
#if CC_UPD_PIPE
        issue();
#endif
    }
    if (n) {
        reinterpret_cast<double2*>(st)[0] = make_double2(s.V, s.c);
        reinterpret_cast<double2*>(st)[1] = make_double2(s.last, s.ru);
    }
    if (CC_TIMING_PROBES && dbg_info) {
        // nmax | max slow steps of a lane << 16 | lanes with slow steps << 32 | spikes << 48
        const unsigned lanes_slow = __popc(__ballot_sync(0xffffffffu, dbg_slow > 0));
        const unsigned nspk = __popc(__ballot_sync(0xffffffffu, dbg_spk > 0));
        *dbg_info = (unsigned long long)nmax | ((unsigned long long)warp_max_u32(dbg_slow) << 16) |
                    ((unsigned long long)lanes_slow << 32) | ((unsigned long long)nspk << 48);
    }
}

// Phase A proper: persistent warps claim work items from the queue.
// 6 blocks of 4 warps per SM: 80 registers per thread (no spills) and, with
// HCAP 288, 9,008 B of staging buffer per warp.  24 instead of 20 resident
// warps: config 1 -1.5 %, config 3 and the 33 Hz stress point -6 % per step.
#ifndef CC_STAGE_MINB
#define CC_STAGE_MINB 6
#endif
// PLAN: the planning pass runs at the start of the kernel (its own instantiation,
// so that the separate-k_plan kernel does not carry the planning code).
template <bool PLAN>
__global__ void __launch_bounds__(32 * STAGE_WARPS, CC_STAGE_MINB)
k_stage(const cc_shard sh) {
    extern __shared__ __align__(16) char nsm[];
    cc_ctl* ctl = sh.ctl;
    const long long t = *(volatile long long*)&ctl->t;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    StageBuf B = carve(nsm + wib * stage_warp_bytes());
    if (threadIdx.x == 0) x_pushed_block() = 0;       // (published by the barriers below)
    __shared__ double2 s_xt[32];                      // 2^(j/32) table of fexp
    if (threadIdx.x < 32) s_xt[threadIdx.x] = c_exp2_tab[threadIdx.x];
    const int t_mod_l = (int)pos_mod(t, sh.log_slots);
    const uint32_t K = (uint32_t)sh.bin_cap;
    const double t0 = (double)t * sh.dt;
    const double inv_dt = 1.0 / sh.dt;
    // planning phase (k_plan's work, one group per warp per round), then a
    // grid-wide barrier: the persistent grid is co-resident (cooperative launch).
    // Chosen by cc_neuron_step when there are more groups than warps: k_plan's
    // separate, 48-warps-per-SM grid is faster for a single round (config 1).
    if constexpr (PLAN) {
        const int rounds = (sh.n_groups + (int)(gridDim.x * STAGE_WARPS) - 1)
                           / (int)(gridDim.x * STAGE_WARPS);
        for (int r = 0; r < rounds; ++r)
            plan_group(sh, t, (r * (int)gridDim.x + (int)blockIdx.x) * STAGE_WARPS + wib);
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(&sh.tailc[64], 1u);
            unsigned spins = 0;
            while (*(volatile unsigned*)&sh.tailc[64] < gridDim.x) {
                __nanosleep(64);
                if (++spins == (1u << 24)) { cc_raise(ctl, CC_ERR_GRIDSYNC, t); break; }
            }
            __threadfence();
        }
        __syncthreads();
    }
    // step t+1's delay >= 2 units (spikes of steps t-1 .. t+1-d_max, all
    // logged): offered to the warps that run out of work items
    // (block-wide unit tables behind the warps' staging buffers: d_max and
    // d_max + 1 words, stage_tail_bytes())
    const int D = sh.d_max;
    unsigned* const a_n = reinterpret_cast<unsigned*>(nsm + STAGE_WARPS * stage_warp_bytes());
    unsigned* const a_pre = a_n + D;
    const bool tail_deliver = D > 1 && !(sh.flags & CC_FLAG_NO_TAIL_DELIVERY) && !sh.l1_ncnt;
    if (tail_deliver) unit_prefix(sh, slot_add(t_mod_l, 1, sh.log_slots), D - 1, a_n, a_pre);
    // queued items per size class (k_plan is complete); claimed largest first
    __shared__ unsigned cls_n[CC_ITEM_CLASSES];
    if (threadIdx.x < CC_ITEM_CLASSES)
        cls_n[threadIdx.x] = min(*(volatile unsigned*)&ctl->cls_n[threadIdx.x],
                                 (unsigned)sh.round_cap);
    __syncthreads();
    unsigned n_items = 0;
    for (int c = 0; c < CC_ITEM_CLASSES; ++c) n_items += cls_n[c];
    if (*(volatile unsigned*)&ctl->error_bits) n_items = 0u;
    uint32_t my_spikes = 0;
    // first item of every warp by its index (no burst of same-address claims
    // at kernel start), the rest claimed in order after them
    const unsigned n_stage_warps = gridDim.x * STAGE_WARPS;
    bool first = CC_STATIC_FIRST != 0;
    for (;;) {
        unsigned item = 0;
        if (first) {
            item = blockIdx.x * STAGE_WARPS + wib;
            first = false;
        } else {
            if (lane == 0)
#if CC_CLAIM_OWN_LINE
                item = atomicAdd(&sh.tailc[96], 1u) + (CC_STATIC_FIRST ? n_stage_warps : 0u);
#else
                item = atomicAdd(&ctl->round_next, 1u) + (CC_STATIC_FIRST ? n_stage_warps : 0u);
#endif
            item = __shfl_sync(0xffffffffu, item, 0);
        }
        if (item >= n_items) break;
        CC_DBG(0, gtimer());
        CC_DBG(5, 0ull);
        unsigned r = item;                        // class c, position r in it
        int c = 0;
        while (r >= cls_n[c]) r -= cls_n[c++];    // terminates: item < n_items
        const size_t q = (size_t)c * sh.round_cap + r;
        const int group = (int)sh.rounds[2 * q];
        const uint32_t lr = sh.rounds[2 * q + 1];
        const int l0 = (int)(lr & 0xff), l1 = (int)(lr >> 8);
        const int li0 = group * 32;
        const int li = li0 + lane;
        const bool in = lane >= l0 && lane < l1 && li < sh.n_local;
        uint32_t n = 0, n_r = 0, gid = 0;
        if (in) {
            n = (uint32_t)sh.ev_n[li];
            n_r = (uint32_t)sh.ev_nr[li];
            gid = sh.gid[li];
            const double2 b = reinterpret_cast<const double2*>(sh.state + (size_t)li * 4)[1];
            const double c = sh.state[(size_t)li * 4 + 1];
            B.o_last[lane] = b.x;
            B.o_ru[lane] = b.y;
            B.o_flag[lane] = (uint32_t)neuron_pop(sh, gid) | (c != 0.0 ? 2u : 0u);
        }
        const uint32_t n_e = n - min(n, n_r);
        const uint32_t nb = min(n_r, K);
        const bool go = in && n > 0;
        uint32_t rtot;
        const uint32_t roff = warp_excl_scan(go ? n : 0u, rtot);
        B.seg[lane] = (int)roff;
        if (lane == 31) B.seg[32] = (int)rtot;
        // Phases 1-3 of the item, instantiated twice: with the warp's shared-
        // memory buffer (every item of <= NEURON_WCAP inputs: the hot path,
        // shared-memory addressing only), and with a global-scratch buffer for a
        // single neuron larger than that (an item of its own; onset bursts).
        // Returns false if a capacity error was raised.
        auto stage = [&](auto spill_tag) -> bool {
        constexpr bool SPILL = decltype(spill_tag)::value;
        double* Et = B.t; uint32_t* Es = B.src; float* Ew = B.w; uint16_t* Ep = B.perm;
        uint32_t* Ek = B.keep;
        uint16_t* Epv = B.prov;
        uint8_t* Eo = B.own;
        uint8_t* Eq = B.owns;
        if constexpr (SPILL) {
            // a single neuron larger than the shared buffer: stage in global scratch
            unsigned long long at = 0;
            int ok = 1;
            if (lane == 0) {
                if (rtot > 65535u) ok = 0;
                at = atomicAdd(&ctl->scratch_used, (unsigned long long)rtot);
                if (at + rtot > (unsigned long long)sh.scratch_cap) ok = 0;
                if (!ok) cc_raise(ctl, CC_ERR_SCRATCH, t);
                atomicAdd(&ctl->spilled_total, 1ull);
            }
            ok = __shfl_sync(0xffffffffu, ok, 0);
            at = __shfl_sync(0xffffffffu, at, 0);
            if (!ok) return false;
            // spill layout: 3 words of 8 B per event (t, src|w, keep|perm|own)
            double* base = reinterpret_cast<double*>(sh.scratch) + at * 3;
            const uint32_t cap = rtot;
            Et = base;
            Es = reinterpret_cast<uint32_t*>(base + cap);
            Ew = reinterpret_cast<float*>(Es + cap);
            Ek = reinterpret_cast<uint32_t*>(base + 2 * cap);
            Ep = reinterpret_cast<uint16_t*>(Ek + cap);
            Eo = reinterpret_cast<uint8_t*>(Ep + cap);
            Eq = Eo + cap;
            Epv = reinterpret_cast<uint16_t*>(reinterpret_cast<double*>(sh.scratch)
                                              + 6ull * sh.scratch_cap + at);
        }
        __syncwarp();
        // ---- 1a gather this slot's records of the group (contiguous list, then
        //      the group's run of the grouped overflow), keep the item's lanes
        {
            const uint32_t c_all = sh.grp_n[group];
            // lane j < NSUB: records kept in sub-list j
            const uint32_t cj = lane < NSUB ? sh.grp_sub[(size_t)group * NSUB + lane] : 0u;
            uint32_t c_list = cj;
#pragma unroll
            for (int o = NSUB >> 1; o > 0; o >>= 1) c_list += __shfl_xor_sync(0xffffffffu, c_list, o);
            c_list = __shfl_sync(0xffffffffu, c_list, 0);
            const size_t KS = (size_t)K + sh.bin_pad;
            const uint64_t* lst = list_set(sh, t).rec + (size_t)group * NSUB * KS;
            const uint4* ov = reinterpret_cast<const uint4*>(sh.ovf_sorted) + sh.ovf_off[group];
            B.hist[lane] = 0u;                          // per-lane fill cursors
            __syncwarp();
            auto keep = [&](uint64_t rec) {             // stage a record of the item's lanes
                const int L = (int)((uint32_t)rec & 31u);
                if (L < l0 || L >= l1) return;
                const int dst = B.seg[L] + (int)atomicAdd(&B.hist[L], 1u);
                CC_CHK(ctl, dst >= B.seg[L] && dst < B.seg[L + 1] && dst < (int)rtot);
                const Ev ev = make_rec_event(sh, rec, t_mod_l);
                Et[dst] = ev.t; Es[dst] = ev.src; Ew[dst] = ev.w;
                Eo[dst] = (uint8_t)L;
            };
            // the sub-lists the item's lanes [l0, l1) fall into (sub-lists by
            // lane range), one after the other, four records per lane in flight
            int j0 = 0, j1 = NSUB;
#if CC_SUB_BY_LANE
            if (NSUB > 1) {
                j0 = (l0 * NSUB) >> 5;
                j1 = (((l1 - 1) * NSUB) >> 5) + 1;
            }
#endif
            for (int j = j0; j < j1; ++j) {
                const uint32_t cnt = __shfl_sync(0xffffffffu, cj, j);
                const uint64_t* lj = lst + (size_t)j * KS;
                for (uint32_t r0 = 0; r0 < cnt; r0 += 128) {
                    uint64_t rec[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t q0 = r0 + u * 32 + lane;
                        rec[u] = q0 < cnt ? lj[q0] : ~0ull;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (rec[u] != ~0ull) keep(rec[u]);
                }
            }
            // then the group's run of the grouped overflow list
            for (uint32_t q0 = lane; q0 < c_all - c_list; q0 += 32) {
                const uint4 q = ov[q0];
                keep((uint64_t)((q.z << 5) | q.y) | ((uint64_t)q.w << 32));
            }
            __syncwarp();
        }
        // ---- 1b external drive: event times (t_step + u) * dt with
        //      u = counter_uniforms(EXTERNAL_TIME, gid, t, j) (engine.py:191-206),
        //      flattened over the warp (lane owner map in the idle prov buffer)
        {
            const uint32_t ne = go ? n_e : 0u;
            uint32_t etot;
            const uint32_t eoff = warp_excl_scan(ne, etot);
            const uint64_t h4 = ne ? cc_splitmix64(cc_splitmix64(sh.h2_time ^ (uint64_t)gid)
                                                   ^ (uint64_t)t) : 0ull;
            if constexpr (!SPILL) {
                uint64_t* hq = reinterpret_cast<uint64_t*>(B.hist + 32);   // [32], idle here
                uint32_t* eo = B.hist + 96;
                uint32_t* eb = B.hist + 128;
                uint8_t* own = reinterpret_cast<uint8_t*>(B.prov);
                hq[lane] = h4;
                eo[lane] = eoff;
                eb[lane] = roff + n_r;
                for (uint32_t k = 0; k < ne; ++k) own[eoff + k] = (uint8_t)lane;
                __syncwarp();
                for (uint32_t f = lane; f < etot; f += 32) {
                    const int L = own[f];
                    const uint32_t k = f - eo[L];
                    const int dst = (int)(eb[L] + k);
                    Et[dst] = ((double)t + cc_u53(cc_splitmix64(hq[L] ^ (uint64_t)k))) * sh.dt;
                    Es[dst] = CC_EXT_SRC;
                    Ew[dst] = 0.0f;
                    Eo[dst] = (uint8_t)L;
                }
            } else {                                    // spilled item: per lane
                const int b0 = (int)roff;
                for (uint32_t k = 0; k < ne; ++k) {
                    Et[b0 + n_r + k] = ((double)t + cc_u53(cc_splitmix64(h4 ^ (uint64_t)k))) * sh.dt;
                    Es[b0 + n_r + k] = CC_EXT_SRC;
                    Ew[b0 + n_r + k] = 0.0f;
                    Eo[b0 + n_r + k] = (uint8_t)lane;
                }
            }
        }
        CC_DBG(1, gtimer());
        // ---- 2 order each neuron's inputs by (t, src): counting sort on a
        //      monotone time bucket (adaptive count per neuron, flattened over
        //      the warp), then the exact rank of each input inside its bucket
        {
            const uint32_t nbl = go ? min(2u * n, (uint32_t)(HCAP - 32) * n / rtot + 1u) : 0u;
            uint32_t nbt;
            const uint32_t cb = warp_excl_scan(nbl, nbt);
            B.cbk[lane] = cb | (nbl << 16);
            B.bsc[lane] = (double)nbl * inv_dt;      // any monotone map of t will do
            __syncwarp();
            for (uint32_t i = lane; i < nbt; i += 32) B.hist[i] = 0u;
            __syncwarp();
            for (uint32_t e = lane; e < rtot; e += 32) {
                const uint32_t o = Eo[e];
                const uint32_t ck = B.cbk[o];
                const int b = min(max(__double2int_rz((Et[e] - t0) * B.bsc[o]), 0),
                                  (int)(ck >> 16) - 1);
                const uint32_t key = (ck & 0xffffu) + (uint32_t)b;
                CC_CHK(ctl, key < nbt && nbt <= (uint32_t)HCAP);
                Ek[e] = (key << 16) | atomicAdd(&B.hist[key], 1u);
            }
            __syncwarp();
            // exclusive scan of the flattened counters: bucket starts, which
            // are already segmented by neuron (lane-major order); packed
            // start | count << 16
            const uint32_t per = ((nbt + 31u) / 32u) | 1u;      // odd: lane chunks hit distinct banks
            const uint32_t i0 = min(lane * per, nbt), i1 = min(i0 + per, nbt);
            uint32_t sum = 0;
            for (uint32_t i = i0; i < i1; ++i) sum += B.hist[i];
            uint32_t tot2;
            uint32_t base = warp_excl_scan(sum, tot2);
            for (uint32_t i = i0; i < i1; ++i) {
                const uint32_t c = B.hist[i];
                B.hist[i] = base | (c << 16);
                base += c;
            }
            __syncwarp();
            // scatter: singleton buckets are final, others provisional
            for (uint32_t e = lane; e < rtot; e += 32) {
                const uint32_t kp = Ek[e];
                const uint32_t h = B.hist[kp >> 16];
                const uint32_t o = Eo[e];
                const uint32_t rel = e - (uint32_t)B.seg[o];
                const uint32_t pos = (h & 0xffffu) + (kp & 0xffffu);
                if ((h >> 16) == 1u) Ep[pos] = (uint16_t)rel;
                else Epv[pos] = (uint16_t)rel;
                Eq[pos] = (uint8_t)o;                   // owner of each sorted slot
            }
            __syncwarp();
            // exact order inside shared buckets: rank among the bucket's inputs
            // by (t, src, w) like lexsort((w, src, tm, tgt)) (engine.py:386);
            // ties by staging index (identical inputs commute)
            for (uint32_t e = lane; e < rtot; e += 32) {
                const uint32_t kp = Ek[e];
                const uint32_t h = B.hist[kp >> 16];
                const uint32_t c = h >> 16;
                if (c == 1u) continue;
                const uint32_t s0 = h & 0xffffu;
                const uint32_t o = Eo[e];
                const int a = B.seg[o];
                const uint32_t rel = e - (uint32_t)a;
                const double te = Et[e];
                const uint32_t se = Es[e];
                const float we = Ew[e];
                uint32_t rank = 0;
                for (uint32_t q = s0; q < s0 + c; ++q) {
                    const uint32_t pq = Epv[q];
                    const double tq = Et[a + pq];
                    rank += tq < te ? 1u : 0u;
                    if (tq == te && pq != rel) {        // rare: equal times
                        const uint32_t sq = Es[a + pq];
                        const float wq = Ew[a + pq];
                        rank += (sq < se || (sq == se && (wq < we || (wq == we && pq < rel))))
                                    ? 1u : 0u;
                    }
                }
                Ep[s0 + rank] = (uint16_t)rel;
            }
        }
        __syncwarp();
        CC_DBG(2, gtimer());
        // ---- 3 decay factors of every input (flattened over the warp), valid
        //      under the step-start refractory window and fatigue flag, written
        //      with t and w as one ordered record per input
        unsigned long long rbase = 0;
        if (lane == 0 && rtot) {
#if CC_CLAIM_OWN_LINE
            rbase = atomicAdd(&sh.tailc[128], rtot);     // own L2 line
#else
            rbase = atomicAdd(&ctl->stream_used, (unsigned long long)rtot);
#endif
            // evrec_cap covers a step's expected list capacity + overflow + drive
            if (rbase + rtot > (unsigned long long)sh.evrec_cap) cc_raise(ctl, CC_ERR_EVREC, t);
        }
        rbase = __shfl_sync(0xffffffffu, rbase, 0);
        if (rbase + rtot > (unsigned long long)sh.evrec_cap) return false;
        {
            double2* R = reinterpret_cast<double2*>(sh.evrec) + 3 * rbase;
            for (uint32_t p = lane; p < rtot; p += 32) {
                const int o = Eq[p];
                const int a = B.seg[o];
                const int e = a + Ep[p];
                const double te = Et[e];
                const double last = (int)p == a ? B.o_last[o] : Et[a + Ep[p - 1]];
                const double ru = B.o_ru[o];
                const uint32_t fl = B.o_flag[o];
                const double ff = fmin(fmax(last, ru), te);
                double em, ec, f;
                const cc_pop& P = sh.pop[fl & 1u];
                decay_factors(P, te - ff, (fl & 2u) != 0, em, ec, f, s_xt);
                // fatigue decay over the refractory part of the gap (slow_step)
#if CC_STAGE_ECR
                const double ecr = (ff != last && (fl & 2u))
                                       ? fexp(-div_rn(ff - last, P.tau_c, P.r_tau_c), s_xt) : 1.0;
#else
                const double ecr = 1.0;         // (computed by slow_step when it is needed)
#endif
                const double wv = (Es[e] == CC_EXT_SRC) ? sh.ext_weight : (double)Ew[e];
#if CC_EVREC_STREAM
                __stcs(R + 3 * p, make_double2(te, wv));
                __stcs(R + 3 * p + 1, make_double2(em, ec));
                __stcs(R + 3 * p + 2, make_double2(f, ecr));
#else
                R[3 * p] = make_double2(te, wv);
                R[3 * p + 1] = make_double2(em, ec);
                R[3 * p + 2] = make_double2(f, ecr);
#endif
            }
        }
        if (go) sh.ev_off[li] = (int32_t)(rbase + roff);
        CC_DBG(3, gtimer());
        return true;
        };
        if (!(rtot > (uint32_t)NEURON_WCAP ? stage(std::true_type{}) : stage(std::false_type{})))
            continue;
        // ---- 4 publish; the warp finishing a group's last item runs the
        //      group's in-order update (one lane per neuron)
        __threadfence();
        unsigned prev = 0;
        if (lane == 0) prev = atomicAdd(&sh.grp_done[group], 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev + 1u == sh.grp_items[group]) {
            __threadfence();
            if (lane == 0) sh.grp_done[group] = 0u;
            CC_DBG(5, gtimer());                       // update start (0: no update)
            unsigned long long dbg_info = 0ull;
            update_group(sh, li0, t, t_mod_l, reinterpret_cast<double2*>(nsm + wib * stage_warp_bytes()),
                         my_spikes, s_xt, &dbg_info);
            CC_DBG(1, dbg_info | (1ull << 63));        // (probe runs: overwrites "gathered")
        }
        {
            CC_DBG(4, gtimer());
            CC_DBG(6, (unsigned long long)rtot);
            CC_DBG(7, (unsigned long long)(blockIdx.x * STAGE_WARPS + wib));
        }
    }
    // ---- 5 tail: deliver step t+1's delay >= 2 units (claimed in order from
    //      tailc[0]; k_deliver(t+1) delivers the ones left and the delay-1
    //      units) while the last items and group updates finish
    // Claims stop once every warp is out of items (the step's own work is
    // done): the rest goes to k_deliver(t+1), whose pipelined grid is faster.
    unsigned idle_prev = 0;
    unsigned long long tail_ev = 0;
    if (lane == 0) idle_prev = atomicAdd(&sh.tailc[32], 1u);
    // (stop at CC_TAIL_STOP/16 of the warps idle: units in flight past the
    // step's last update lengthen the kernel)
    const unsigned n_warps = gridDim.x * STAGE_WARPS * CC_TAIL_STOP / 16;
    if (tail_deliver && __shfl_sync(0xffffffffu, idle_prev, 0) + 1u < n_warps &&
        !*(volatile unsigned*)&ctl->error_bits) {
        const unsigned n_a = a_pre[D - 1];
        const int t1_mod = slot_add(t_mod_l, 1, sh.log_slots);
        const ListSet S1 = list_set(sh, t + 1);
        constexpr int UT = 8;
        int kc = 0;
        for (;;) {
            unsigned u = n_a;
            if (lane == 0 && *(volatile unsigned*)&sh.tailc[32] < n_warps)
                u = atomicAdd(&sh.tailc[0], 1u);
            u = __shfl_sync(0xffffffffu, u, 0);
            if (u >= n_a) break;
            uint64_t st;
            uint32_t ln, rf;
            unit_desc(sh, t1_mod, a_n, a_pre, u, kc, st, ln, rf);
            if ((lane & (del_lps(sh) - 1)) == 0) tail_ev += ln;      // one lane per spike
            const uint32_t lmax = warp_max_u32(ln);
            for (int p = 0; (uint32_t)(p * del_lps(sh) * UT) < lmax; ++p) {
                int tg[UT];
                float w[UT];
                load_pass<UT>(sh, st, ln, p, tg, w);
                deposit_pass<UT>(sh, S1, kc % NSUB, tg, w, rf, t + 1);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tail_ev += __shfl_xor_sync(0xffffffffu, tail_ev, o);
    if (lane == 0 && tail_ev) atomicAdd(&ctl->tail_events, tail_ev);
    // spike counter: one atomic per block; last block out retires the step
    unsigned s_sum = my_spikes;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
    __shared__ unsigned blk_s;
    if (threadIdx.x == 0) blk_s = 0;
    __syncthreads();
    if (lane == 0 && s_sum) atomicAdd(&blk_s, s_sum);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blk_s) atomicAdd(&ctl->n_spikes, (unsigned long long)blk_s);
        // (peer exchange: the block's pushes to other GPUs are ordered before
        // its completion, which the last block's release publishes)
        if (sh.xdst && x_pushed_block()) __threadfence_system(); else __threadfence();
        if (atomicAdd(&ctl->done_stage, 1u) == gridDim.x - 1) {
            ctl->done_stage = 0;
            sh.tailc[32] = 0u;
            ctl->stream_used = sh.tailc[128];  // records used this step (diagnostics)
            sh.ovf_cnt[t & 1] = 0;             // step t's inputs fully consumed
            if (sh.xdst) x_publish(sh.xdst, sh.xcnt, sh.n_ranks, ctl, t);
            __threadfence();
            *(volatile long long*)&ctl->t = t + 1;
        }
    }
}

// ------------------------------------------------------------------ k_probe
// Probe recording (tests only): state of the probed neurons after step t and
// V advanced to (t+1)*dt on a copy, the harness of oracle/make_golden.py.
__global__ void k_probe(const cc_shard sh) {
    const long long t = *(volatile long long*)&sh.ctl->t - 1;
    const int li = blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= sh.n_local || t < 0 || t >= sh.probe_steps) return;
    const int ps = sh.probe_map[li];
    if (ps < 0) return;
    const double* st = sh.state + (size_t)li * 4;
    NState s{st[0], st[1], st[2], st[3]};
    double* o = sh.probe_out + ((size_t)t * sh.n_probe + ps) * 5;
    o[0] = s.V; o[1] = s.c; o[2] = s.last; o[3] = s.ru;
    advance(s, sh.pop[neuron_pop(sh, sh.gid[li])], (double)(t + 1) * sh.dt);
    o[4] = s.V;
}

// Counting sort of one slot's overflow records by target, by a single block
// (only runs in steps that overflowed the dense bins).
__device__ void group_overflow(const cc_shard& sh, const ListSet& S, unsigned m) {
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry;
    const int n = sh.n_groups;
    const uint32_t K = (uint32_t)sh.bin_cap;
    const uint32_t* cnt = S.cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + threadIdx.x;
        uint32_t v = 0u;
        if (i < n) {
#pragma unroll
            for (int j = 0; j < NSUB; ++j) {
                const uint32_t c = cnt[((size_t)i * NSUB + j) * CC_CNT_STRIDE];
                v += c > K ? c - K : 0u;
            }
        }
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = lane < nwarp ? wsum[lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            if (lane < nwarp) wsum[lane] = w;
        }
        __syncthreads();
        const uint32_t before = carry + (warp ? wsum[warp - 1] : 0u) + x - v;
        if (i < n) sh.ovf_off[i] = (int32_t)before;
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[nwarp - 1];
        __syncthreads();
    }
    const uint4* rec = S.ovf;
    uint4* out = reinterpret_cast<uint4*>(sh.ovf_sorted);
    for (unsigned j = threadIdx.x; j < m; j += blockDim.x) {
        const uint4 r = rec[j];
        const long long p = (long long)sh.ovf_off[r.x] + atomicAdd(&sh.ovf_fill[r.x], 1);
        if (p < sh.ovf_cap) out[p] = r;       // beyond: records were dropped, error raised
    }
    __syncthreads();
    for (unsigned j = threadIdx.x; j < m; j += blockDim.x) sh.ovf_fill[rec[j].x] = 0;
}

// Per-step bookkeeping of the first delivery kernel's first thread.
__device__ __forceinline__ void deliver_prologue(const cc_shard& sh, long long t) {
    cc_ctl* ctl = sh.ctl;
    const int L = sh.log_slots;
    // recurrent_events: row lengths of the spikes of step t - 1, counted at
    // their expansion step like engine.py:366
    const unsigned long long ev = sh.log_len[pos_mod(t - 1, L)];
    if (ev) atomicAdd(&ctl->rec_events, ev);
    sh.log_ctr[pos_mod(t, L)] = 0ull;      // the slot k_stage(t) fills (step t - d_max - 1)
    sh.tailc[64] = 0u;                     // k_stage(t)'s grid barrier
    sh.log_len[pos_mod(t, L)] = 0ull;
    ctl->scratch_used = 0ull;
    ctl->stream_used = 0ull;
    sh.tailc[128] = 0u;                    // k_stage's ordered-input record cursor
    ctl->n_rounds = 0u;
    ctl->round_next = 0u;
    sh.tailc[96] = 0u;                     // k_stage's item claims (own L2 line)
#pragma unroll
    for (int c = 0; c < CC_ITEM_CLASSES; ++c) ctl->cls_n[c] = 0u;
}

// Block-wide end of the step's last delivery kernel: the deposited-event count
// and, in the last block out (step t's inputs are complete then), the overflow
// records grouped by group for k_plan(t).
__device__ __forceinline__ void deliver_epilogue(const cc_shard& sh, const ListSet& S,
                                                 unsigned long long my_ev) {
    cc_ctl* ctl = sh.ctl;
    const int lane = threadIdx.x & 31;
    __shared__ bool am_last;
    __shared__ unsigned long long blk_ev;
    if (threadIdx.x == 0) blk_ev = 0ull;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_ev += __shfl_xor_sync(0xffffffffu, my_ev, o);
    if (lane == 0 && my_ev) atomicAdd(&blk_ev, my_ev);
    __syncthreads();
    if (threadIdx.x == 0 && blk_ev) atomicAdd(&ctl->del_events, blk_ev);
    if (threadIdx.x == 0) {
        __threadfence();
        am_last = atomicAdd(&ctl->done_deliver, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (CC_TIMING_PROBES && (sh.flags & 256) && threadIdx.x == 0) {
        unsigned long long* d_ = reinterpret_cast<unsigned long long*>(sh.scratch)
                                 + (size_t)sh.scratch_cap * 7 - 65536ull * 8 - 65536ull * 4 - (size_t)(blockIdx.x + 1);
        d_[0] = gtimer();
    }
    if (!am_last) return;
    __threadfence();
    const unsigned m = min(*(volatile unsigned*)S.ovf_cnt, (unsigned)sh.ovf_cap);
    if (threadIdx.x == 0) {
        ctl->done_deliver = 0;
        ctl->ovf_grouped = m;
        sh.tailc[0] = 0u;                      // k_stage(t) offers step t+1's units
    }
    if (m == 0) return;
    group_overflow(sh, S, m);
}

// Delivery of arrival step t (pull): the events arriving at t are the delay-d
// segments of the rows of the spikes of step t - d, d = 1..d_max.  The units
// of delay >= 2 were already offered to the idle warps of k_stage(t - 1)
// (tailc[0] counts the ones they claimed); this kernel delivers the rest
// and the delay-1 units, software-pipelined (the next pass's or unit's CSR
// loads are issued before this pass's reservations and deposits).
__global__ void __launch_bounds__(CC_DEL_THREADS, CC_DEL_MINB)
k_deliver(const cc_shard sh) {
    const unsigned long long dbg_t0 = gtimer();
    cc_ctl* ctl = sh.ctl;
    const long long t = *(volatile long long*)&ctl->t;
    if (*(volatile unsigned*)&ctl->error_bits) return;      // failed run: stop working
    const int L = sh.log_slots, D = sh.d_max;
    __shared__ unsigned s_n[DEL_DMAX], s_pre[DEL_DMAX + 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) deliver_prologue(sh, t);
    // units [0, c) were delivered by k_stage(t - 1)'s idle warps (claimed in
    // order); read by warp 1 while warp 0 builds the unit prefix
    __shared__ unsigned s_c0;
    if (threadIdx.x == 32) s_c0 = *(volatile unsigned*)&sh.tailc[0];
    const int t_mod = (int)pos_mod(t, L);
    unit_prefix(sh, t_mod, D, s_n, s_pre);
    const unsigned n_units = s_pre[D];
    const unsigned c0 = min(s_c0, s_pre[D - 1]);
    const ListSet S = list_set(sh, t);
    const int lane = threadIdx.x & 31;
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    const unsigned long long dbg_t1 = gtimer();
    constexpr int U = CC_DEL_U;
    const int SPAN = del_lps(sh) * U;                        // synapses per spike per pass
    int kc = 0;
    unsigned u = c0 + wid;
    uint64_t st = 0, stn = 0;
    uint32_t ln = 0, rf = 0, lnn = 0, rfn = 0;
    int kcur = 0, kn = 0;
    if (u < n_units) { unit_desc(sh, t_mod, s_n, s_pre, u, kc, st, ln, rf); kcur = kc; }
    if (u + nw < n_units) { unit_desc(sh, t_mod, s_n, s_pre, u + nw, kc, stn, lnn, rfn); kn = kc; }
    uint32_t lmax = warp_max_u32(ln);
    int p = 0;
    int tg[U];
    float w[U];
    if (u < n_units) load_pass<U>(sh, st, ln, 0, tg, w);
    const bool cnt_lane = (lane & (del_lps(sh) - 1)) == 0;   // one lane per spike counts
    unsigned long long my_ev = (u < n_units && cnt_lane) ? ln : 0u;
    while (u < n_units) {
        // next pass of this unit, else the first pass of the warp's next unit
        unsigned u2 = u;
        int p2 = p + 1;
        uint64_t st2 = st;
        uint32_t ln2 = ln, rf2 = rf, lmax2 = lmax;
        int k2 = kcur;
        const bool adv = (uint32_t)(p2 * SPAN) >= lmax;
        if (adv) {
            u2 = u + nw; p2 = 0; st2 = stn; ln2 = lnn; rf2 = rfn; k2 = kn;
            lmax2 = warp_max_u32(lnn);
        }
        int tg2[U];
        float w2[U];
        if (u2 < n_units) load_pass<U>(sh, st2, ln2, p2, tg2, w2);
        else {
#pragma unroll
            for (int k = 0; k < U; ++k) tg2[k] = -1;
        }
        if (adv && u2 + nw < n_units) { unit_desc(sh, t_mod, s_n, s_pre, u2 + nw, kc, stn, lnn, rfn); kn = kc; }
        if (adv && u2 < n_units && cnt_lane) my_ev += ln2;
        deposit_pass<U>(sh, S, kcur % NSUB, tg, w, rf, t);
#pragma unroll
        for (int k = 0; k < U; ++k) { tg[k] = tg2[k]; w[k] = w2[k]; }
        u = u2; p = p2; st = st2; ln = ln2; rf = rf2; lmax = lmax2; kcur = k2;
    }
    if (CC_TIMING_PROBES && (sh.flags & 256) && lane == 0) {
        unsigned long long* d_ = reinterpret_cast<unsigned long long*>(sh.scratch)
                                 + (size_t)sh.scratch_cap * 7 - 65536ull * 8 - (size_t)(wid + 1) * 4;
        unsigned smid_;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid_));
        d_[0] = dbg_t0; d_[1] = dbg_t1; d_[2] = gtimer();
        d_[3] = (unsigned long long)smid_ | ((unsigned long long)(n_units - c0) << 32);
    }

    // Step t's inputs are complete now (this kernel is their last depositor)
    deliver_epilogue(sh, S, my_ev);
}

#include "route_kernels.cuh"

// Delay-segment table: dseg[r][d] = synapses of row r with delay <= d,
// d = 0..d_max (rows sorted by delay).  One warp per row.
__global__ void k_build_dseg(const int64_t* row_off, const uint8_t* syn_d, int64_t n_rows,
                             int d_max, int stride, uint16_t* out, unsigned* err) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows;
         r += nwarp) {
        const int64_t a = row_off[r];
        const int64_t len = row_off[r + 1] - a;
        uint16_t* o = out + (size_t)r * stride;
        if (len > 65535) {
            if (lane == 0) atomicOr(err, CC_ERR_DSEG);
            continue;
        }
        // delay d starts at the first j with syn_d[j] >= d: lane j writes
        // o[d] = j for d in (syn_d[j-1], syn_d[j]]; the rest is len
        for (int64_t j = lane; j < len; j += 32) {
            const int dj = syn_d[a + j];
            const int dp = j ? (int)syn_d[a + j - 1] : 0;
            for (int d = dp; d < dj; ++d) o[d] = (uint16_t)j;
        }
        const int dl = len ? (int)syn_d[a + len - 1] : 0;
        for (int d = dl + lane; d < stride; d += 32) o[d] = (uint16_t)len;
    }
}

// Multi-shard receive: log the AER events of step ctl->t - 1 that have rows here.
__global__ void k_ingest(const cc_shard sh, const uint32_t* in_gid, const double* in_t,
                         const int32_t* in_n) {
    const long long t = *(volatile long long*)&sh.ctl->t - 1;
    const int e_t = (int)pos_mod(t, sh.log_slots);
    const int n = *in_n;
    const int lane = threadIdx.x & 31;
    const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int b = w0 * 32; b < n; b += nw * 32) {
        const int i = b + lane;
        const bool v = i < n;
        log_spike_warp(sh, t, e_t, v, v ? in_gid[i] : 0u, v ? in_t[i] : 0.0);
    }
}

// Peer exchange, receive half: wait for every linked source's flag of step
// ctl->t - 1 (acquire, system scope), then log its records.
__global__ void __launch_bounds__(256) k_xingest(const cc_shard sh) {
    cc_ctl* ctl = sh.ctl;
    const long long t = *(volatile long long*)&ctl->t - 1;
    const int e_t = (int)pos_mod(t, sh.log_slots);
    // a failed rank stops receiving (its k_stage keeps publishing, so that its
    // peers never wait for it; the hosts agree on the failure per chunk)
    if (*(volatile unsigned*)&ctl->error_bits) return;
    __shared__ uint32_t s_pre[33];
    __shared__ const uint4* s_rec[32];
    if (threadIdx.x < 32) {
        const int s = threadIdx.x;
        uint32_t c = 0;
        const uint4* rec = nullptr;
        if (s < sh.n_ranks) {
            const cc_xpeer& X = sh.xsrc[s];
            if (X.flag[0]) {
                const unsigned long long* f =
                    reinterpret_cast<const unsigned long long*>(X.flag[t & 1]);
                unsigned long long v = ld_acquire_sys(f);
                if ((long long)(v >> 32) < t + 1) {
                    const unsigned long long t0 = gtimer();
                    for (;;) {
                        __nanosleep(128);
                        v = ld_acquire_sys(f);
                        if ((long long)(v >> 32) >= t + 1) break;
                        if ((long long)(gtimer() - t0) > sh.xwait_ns) {
                            cc_raise(ctl, CC_ERR_XWAIT, t);
                            v = 0ull;
                            break;
                        }
                    }
                }
                c = min((uint32_t)v, X.cap);
                rec = reinterpret_cast<const uint4*>(X.rec[t & 1]);
            }
        }
        uint32_t tot;
        const uint32_t ex = warp_excl_scan(c, tot);
        s_pre[s] = ex;
        s_rec[s] = rec;
        if (s == 31) s_pre[32] = tot;
        if (s == 0 && blockIdx.x == 0 && tot) ctl->x_recv += tot;
    }
    __syncthreads();
    const uint32_t total = s_pre[32];
    const int lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    int s = 0;
    for (uint32_t b = w0 * 32; b < total; b += nw * 32) {
        const uint32_t i = b + lane;
        const bool v = i < total;
        uint32_t gid = 0;
        double te = 0.0;
        if (v) {
            while (s_pre[s + 1] <= i) ++s;
            CC_CHK(ctl, s < sh.n_ranks && s_rec[s] != nullptr && i - s_pre[s] < sh.xsrc[s].cap);
            const uint4 r = s_rec[s][i - s_pre[s]];
            gid = r.x;
            te = __longlong_as_double((long long)(((unsigned long long)r.z << 32) | r.y));
        }
        log_spike_warp(sh, t, e_t, v, gid, te);
    }
}

// Multi-shard send (source_masks, network.py:229-230; the counters-then-payloads
// message of deliver_spikes, network.py:325-379, as one fixed-size slot per
// destination): slot d = {count, (gid, t bits) x count}, int64 words.  One block,
// so the per-destination counters live in shared memory; consumes the out-list.
__global__ void __launch_bounds__(1024)
k_pack_aer(const cc_shard sh, const uint32_t* dest_mask, int n_dest, int cap,
           long long* send, const int32_t* local_of_col) {
    __shared__ unsigned cnt[32];
    cc_ctl* ctl = sh.ctl;
    if (threadIdx.x < 32) cnt[threadIdx.x] = 0u;
    __syncthreads();
    const unsigned n = min(*(volatile unsigned*)&ctl->out_n, (unsigned)sh.out_cap);
    const size_t stride = 1 + 2 * (size_t)cap;
    const int n_col = sh.n_col;
    for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t g = sh.out_gid[i];
        const uint32_t li = (uint32_t)local_of_col[g / n_col] * n_col + g % n_col;
        const uint32_t m = dest_mask[li];
        const long long tb = __double_as_longlong(sh.out_t[i]);
        for (int d = 0; d < n_dest; ++d) {
            if (!(m >> d & 1u)) continue;
            const unsigned p = atomicAdd(&cnt[d], 1u);
            if (p < (unsigned)cap) {
                send[d * stride + 1 + 2 * (size_t)p] = (long long)g;
                send[d * stride + 2 + 2 * (size_t)p] = tb;
            } else {
                cc_raise(ctl, CC_ERR_OUTLIST, *(volatile long long*)&ctl->t - 1);
            }
        }
    }
    __syncthreads();
    if ((int)threadIdx.x < n_dest) send[threadIdx.x * stride] = (long long)min(cnt[threadIdx.x], (unsigned)cap);
    if (threadIdx.x == 0) ctl->out_n = 0u;                // out-list consumed
}

// Multi-shard receive of the packed slots of n_src sources: log the AER events
// of step ctl->t - 1 that have rows here (rows_for, network.py:135-141).
__global__ void k_ingest_aer(const cc_shard sh, const long long* recv, int n_src, int cap) {
    const long long t = *(volatile long long*)&sh.ctl->t - 1;
    const int e_t = (int)pos_mod(t, sh.log_slots);
    if (*(volatile unsigned*)&sh.ctl->error_bits) return;
    const size_t stride = 1 + 2 * (size_t)cap;
    __shared__ uint32_t s_pre[33];
    if (threadIdx.x < 32) {
        const int s = threadIdx.x;
        const uint32_t c = s < n_src ? (uint32_t)min(recv[s * stride], (long long)cap) : 0u;
        uint32_t tot;
        const uint32_t ex = warp_excl_scan(c, tot);
        s_pre[s] = ex;
        if (s == 31) s_pre[32] = tot;
    }
    __syncthreads();
    const uint32_t total = s_pre[32];
    const int lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    int s = 0;
    for (uint32_t b = w0 * 32; b < total; b += nw * 32) {
        const uint32_t i = b + lane;
        const bool v = i < total;
        uint32_t gid = 0;
        double te = 0.0;
        if (v) {
            while (s_pre[s + 1] <= i) ++s;
            const long long* r = recv + s * stride + 1 + 2 * (size_t)(i - s_pre[s]);
            gid = (uint32_t)r[0];
            te = __longlong_as_double(r[1]);
        }
        log_spike_warp(sh, t, e_t, v, gid, te);
    }
}

// Test probe of the decay-factor exponentials (tests/test_gpu_parity.py).
__global__ void k_test_math(int kind, const double* x, double* out, int64_t n) {
    __shared__ double2 xt[32];
    if (threadIdx.x < 32) xt[threadIdx.x] = c_exp2_tab[threadIdx.x];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        out[i] = kind == 0 ? fexp(v, xt) : kind == 1 ? fexpm1(v) : kind == 2 ? exp(v) : expm1(v);
    }
}

__global__ void k_init_state(const cc_shard sh) {
    const int li = blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= sh.n_local) return;
    const uint32_t gid = sh.gid[li];
    const int pop = ((int)(gid % (uint32_t)sh.n_col) < sh.n_exc_col) ? 0 : 1;
    const cc_pop& P = sh.pop[pop];
    // counter_uniforms(seed, INIT_STATE, gid, 0, 0)
    const uint64_t h = cc_splitmix64(cc_splitmix64(cc_splitmix64(sh.h2_init ^ (uint64_t)gid)));
    const double u = cc_u53(h);
    double* st = sh.state + (size_t)li * 4;
    reinterpret_cast<double2*>(st)[0] = make_double2(P.V_r + u * (P.V_theta - P.V_r), 0.0);
    reinterpret_cast<double2*>(st)[1] = make_double2(0.0, -INFINITY);
}

}  // namespace

// --------------------------------------------------------------- launchers
extern "C" int cc_set_error(const char* fmt, ...);
extern "C" int cc_check_launch(const char* what);

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

extern "C" int32_t CC_V(cc_sublists)(void) { return CC_SUBLISTS; }

static int stage_blocks_(int d_max, bool fused = false);

// Kernels cc_deliver + cc_neuron_step launch per step for a shard of n_groups
// neuron groups (k_plan runs inside k_stage when groups outnumber its warps).
extern "C" int32_t CC_V(cc_kernels_per_step)(const cc_shard* sh) {
    if (!sh) return 0;
    const bool fused = (sh->flags & CC_FLAG_PLAN_FUSED) ||
                       (!(sh->flags & CC_FLAG_PLAN_SEPARATE) &&
                        sh->n_groups > stage_blocks_(sh->d_max) * STAGE_WARPS);
    return (fused ? 2 : 3) + (sh->l1_cnt ? 1 : 0);
}

extern "C" int CC_V(cc_build_dseg)(const int64_t* row_off, const uint8_t* syn_d, int64_t n_rows,
                             int32_t d_max, int32_t stride, uint16_t* out, unsigned* err,
                             void* stream) {
    if (d_max < 1 || d_max >= DEL_DMAX || stride < d_max + 1 || stride % 8)
        return cc_set_error("cc_build_dseg: need 1 <= d_max < %d, stride >= d_max + 1, "
                            "stride %% 8 == 0", DEL_DMAX);
    if (n_rows <= 0) return 0;
    k_build_dseg<<<sm_count() * 8, 256, 0, (cudaStream_t)stream>>>(row_off, syn_d, n_rows, d_max,
                                                                   stride, out, err);
    return cc_check_launch("k_build_dseg");
}

extern "C" int CC_V(cc_init_state)(const cc_shard* sh, void* stream) {
    if (!sh) return cc_set_error("cc_init_state: null shard");
    if (sh->n_local == 0) return 0;
    k_init_state<<<(sh->n_local + 255) / 256, 256, 0, (cudaStream_t)stream>>>(*sh);
    return cc_check_launch("k_init_state");
}

static int bin_blocks_per_sm = 0;
static int bin_blocks_per_sm_ncnt[CC_L1_NCNT_MAX_RB + 1] = {0};   // with per-neuron counters, by l1_rb
extern "C" int CC_V(cc_prepare)(void);

extern "C" int CC_V(cc_deliver)(const cc_shard* sh, void* stream) {
    if (!sh) return cc_set_error("cc_deliver: null shard");
    if (!sh->l1_cnt) {
        k_deliver<<<sm_count() * CC_DEL_MINB, CC_DEL_THREADS, 0, (cudaStream_t)stream>>>(*sh);
        return cc_check_launch("k_deliver");
    }
    // routed delivery: regions of 2^l1_rb neurons
    if (sh->l1_rb < 5 || sh->l1_rb > 16 || sh->n_regions < 1 ||
        sh->n_regions > CC_L1_MAX_REGIONS ||
        (long long)sh->n_regions << sh->l1_rb < (long long)sh->n_local ||
        (NSUB << (sh->l1_rb - 5)) > CC_L1_MAX_LISTS || sh->l1_cap < 1 ||
        sh->l1_cap >= (1ll << 32) || !sh->l1_ref || !sh->l1_w || !sh->l1_tgt)
        return cc_set_error("cc_deliver: routed delivery needs 5 <= l1_rb <= 16, n_regions = "
                            "ceil(n_local / 2^l1_rb) <= %d, at most %d lists per region, "
                            "l1_cap < 2^32 and the region arrays",
                            CC_L1_MAX_REGIONS, CC_L1_MAX_LISTS);
    if (const int rc = CC_V(cc_prepare)()) return rc;
    k_route<<<CC_RT_BLOCKS ? CC_RT_BLOCKS : sm_count() * CC_RT_MINB, RT_THREADS, route_smem_bytes(),
              (cudaStream_t)stream>>>(*sh);
    if (const int rc = cc_check_launch("k_route")) return rc;
    if (sh->l1_ncnt) {
        if (sh->l1_rb > CC_L1_NCNT_MAX_RB)
            return cc_set_error("cc_deliver: l1_ncnt needs l1_rb <= %d", CC_L1_NCNT_MAX_RB);
        if (!(sh->flags & CC_FLAG_NO_TAIL_DELIVERY))
            return cc_set_error("cc_deliver: l1_ncnt needs CC_FLAG_NO_TAIL_DELIVERY (every list "
                                "record must come through k_bin)");
        k_bin<<<sm_count() * bin_blocks_per_sm_ncnt[sh->l1_rb], BN_THREADS,
                bin_smem_bytes(sh->l1_rb), (cudaStream_t)stream>>>(*sh);
    } else {
        k_bin<<<sm_count() * bin_blocks_per_sm, BN_THREADS, bin_smem_bytes(),
                (cudaStream_t)stream>>>(*sh);
    }
    return cc_check_launch("k_bin");
}

// One-time kernel attributes (not settable inside a CUDA graph capture, so done
// here or on the first eager cc_neuron_step) and the persistent grid size,
// which depends on d_max through the tail tables' share of shared memory.
static bool stage_prepared = false;
static int stage_blocks_by_d[2][DEL_DMAX] = {};        // [planning inside k_stage][d_max]

static size_t stage_smem(int d_max) {
    return stage_warp_bytes() * STAGE_WARPS + stage_tail_bytes(d_max);
}

extern "C" int CC_V(cc_prepare)(void) {
    if (stage_prepared) return 0;
    if (cudaFuncSetAttribute(k_stage<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)stage_smem(DEL_DMAX - 1)) != cudaSuccess ||
        cudaFuncSetAttribute(k_stage<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)stage_smem(DEL_DMAX - 1)) != cudaSuccess)
        return cc_set_error("cc_prepare: %s", cudaGetErrorString(cudaGetLastError()));
    if (cudaFuncSetAttribute(k_route, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)route_smem_bytes()) != cudaSuccess ||
        cudaFuncSetAttribute(k_bin, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)bin_smem_bytes(CC_L1_NCNT_MAX_RB)) != cudaSuccess)
        return cc_set_error("cc_prepare (routed delivery): %s",
                            cudaGetErrorString(cudaGetLastError()));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bin_blocks_per_sm, k_bin, BN_THREADS,
                                                  bin_smem_bytes());
    if (bin_blocks_per_sm < 1) bin_blocks_per_sm = 1;
    for (int rb = 5; rb <= CC_L1_NCNT_MAX_RB; ++rb) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bin_blocks_per_sm_ncnt[rb], k_bin,
                                                      BN_THREADS, bin_smem_bytes(rb));
        if (bin_blocks_per_sm_ncnt[rb] < 1) bin_blocks_per_sm_ncnt[rb] = 1;
    }
    // (filled here, outside any stream capture; the tail tables grow by 16 B
    // per two delay steps, so the occupancy changes at a few d_max values only)
    int per_sm[2] = {0, 0};
    size_t last = 0;
    for (int d = 1; d < DEL_DMAX; ++d) {
        if (stage_smem(d) != last) {
            last = stage_smem(d);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], k_stage<false>,
                                                          32 * STAGE_WARPS, last);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], k_stage<true>,
                                                          32 * STAGE_WARPS, last);
        }
        for (int f = 0; f < 2; ++f)
            stage_blocks_by_d[f][d] = sm_count() * (per_sm[f] > 0 ? per_sm[f] : 1);
    }
    stage_prepared = true;
    return 0;
}

static int stage_blocks_(int d_max, bool fused) {
    CC_V(cc_prepare)();
    return stage_blocks_by_d[fused][d_max < 1 ? 1 : (d_max >= DEL_DMAX ? DEL_DMAX - 1 : d_max)];
}

extern "C" int32_t CC_V(cc_stage_warps)(int32_t d_max) { return stage_blocks_(d_max) * STAGE_WARPS; }

extern "C" int CC_V(cc_neuron_step)(const cc_shard* sh, void* stream) {
    if (!sh) return cc_set_error("cc_neuron_step: null shard");
    if (sh->n_local <= 0) return cc_set_error("cc_neuron_step: empty shard");
    const int groups = (sh->n_local + 31) / 32;
    if (sh->d_max < 1 || sh->d_max >= DEL_DMAX)
        return cc_set_error("cc_neuron_step: d_max must be in [1, %d)", DEL_DMAX);
    const size_t smem = stage_smem(sh->d_max);
    if (const int rc = CC_V(cc_prepare)()) return rc;
    const bool fused = (sh->flags & CC_FLAG_PLAN_FUSED) ||
                       (!(sh->flags & CC_FLAG_PLAN_SEPARATE) &&
                        groups > stage_blocks_(sh->d_max, false) * STAGE_WARPS);
    const int stage_blocks = stage_blocks_(sh->d_max, fused);
    if (!fused) {
        k_plan<<<(groups + 3) / 4, 128, 0, (cudaStream_t)stream>>>(*sh);
        if (const int rc = cc_check_launch("k_plan")) return rc;
        k_stage<false><<<stage_blocks, 32 * STAGE_WARPS, smem, (cudaStream_t)stream>>>(*sh);
    } else {
        // cooperative: the grid barrier after the planning phase needs every
        // block resident (the launch fails instead of hanging otherwise)
        cc_shard s2 = *sh;
        s2.plan_in_stage = 1;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(stage_blocks);
        lc.blockDim = dim3(32 * STAGE_WARPS);
        lc.dynamicSmemBytes = smem;
        lc.stream = (cudaStream_t)stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, k_stage<true>, s2);
    }
    if (const int rc = cc_check_launch("k_stage")) return rc;
    if (sh->n_probe > 0) {
        k_probe<<<(sh->n_local + 255) / 256, 256, 0, (cudaStream_t)stream>>>(*sh);
        if (const int rc = cc_check_launch("k_probe")) return rc;
    }
    return 0;

}

extern "C" int CC_V(cc_ingest)(const cc_shard* sh, const uint32_t* in_gid, const double* in_t,
                         const int32_t* in_n, void* stream) {
    if (!sh) return cc_set_error("cc_ingest: null shard");
    k_ingest<<<sm_count() * 2, 256, 0, (cudaStream_t)stream>>>(*sh, in_gid, in_t, in_n);
    return cc_check_launch("k_ingest");
}

extern "C" int CC_V(cc_pack_aer)(const cc_shard* sh, const uint32_t* dest_mask_by_local,
                           int32_t n_dest, int32_t cap, int64_t* send,
                           const int32_t* local_of_col, void* stream) {
    if (!sh) return cc_set_error("cc_pack_aer: null shard");
    if (n_dest < 1 || n_dest > 32) return cc_set_error("cc_pack_aer: 1..32 shards");
    if (cap < 1) return cc_set_error("cc_pack_aer: cap must be positive");
    k_pack_aer<<<1, 1024, 0, (cudaStream_t)stream>>>(*sh, dest_mask_by_local, n_dest, cap,
                                                     reinterpret_cast<long long*>(send),
                                                     local_of_col);
    return cc_check_launch("k_pack_aer");
}

extern "C" int CC_V(cc_ingest_aer)(const cc_shard* sh, const int64_t* recv, int32_t n_src, int32_t cap,
                             void* stream) {
    if (!sh) return cc_set_error("cc_ingest_aer: null shard");
    k_ingest_aer<<<sm_count(), 256, 0, (cudaStream_t)stream>>>(
        *sh, reinterpret_cast<const long long*>(recv), n_src, cap);
    return cc_check_launch("k_ingest_aer");
}

extern "C" int CC_V(cc_exchange_ingest)(const cc_shard* sh, void* stream) {
    if (!sh) return cc_set_error("cc_exchange_ingest: null shard");
    if (!sh->xsrc || !sh->xdst) return cc_set_error("cc_exchange_ingest: no peer exchange set up");
    if (sh->n_ranks < 1 || sh->n_ranks > 32) return cc_set_error("cc_exchange_ingest: 1..32 ranks");
    // (a step's received spikes are few: a handful of blocks, each waiting on
    // the flags itself, log them)
    k_xingest<<<sm_count() / 4, 256, 0, (cudaStream_t)stream>>>(*sh);
    return cc_check_launch("k_xingest");
}

extern "C" int CC_V(cc_test_math)(int32_t kind, const double* x, double* out, int64_t n, void* stream) {
    if (kind < 0 || kind > 3) return cc_set_error("cc_test_math: kind 0..3");
    if (n <= 0) return 0;
    k_test_math<<<sm_count() * 4, 256, 0, (cudaStream_t)stream>>>(kind, x, out, n);
    return cc_check_launch("k_test_math");
}

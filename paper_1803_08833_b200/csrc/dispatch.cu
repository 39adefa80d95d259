// Public entry points of the step kernels: sim_kernels.cu is compiled once per
// sub-list variant (CC_NSUB_A, CC_NSUB_B sub-lists per 32-neuron group, entry
// points suffixed _s<n>); cc_shard.n_sub selects the variant per shard.
#include "cc_common.cuh"

extern "C" int cc_set_error(const char* fmt, ...);

#define CC_CAT2_(a, b) a##_s##b
#define CC_CAT2(a, b) CC_CAT2_(a, b)
#define A(name) CC_CAT2(name, CC_NSUB_A)
#define B(name) CC_CAT2(name, CC_NSUB_B)
#define CC_DECL(V)                                                                         \
    extern "C" int32_t V(cc_kernels_per_step)(const cc_shard*);                             \
    extern "C" int V(cc_build_dseg)(const int64_t*, const uint8_t*, int64_t, int32_t, int32_t, \
                                    uint16_t*, unsigned*, void*);                           \
    extern "C" int V(cc_init_state)(const cc_shard*, void*);                                \
    extern "C" int V(cc_deliver)(const cc_shard*, void*);                                   \
    extern "C" int V(cc_prepare)(void);                                                     \
    extern "C" int32_t V(cc_stage_warps)(int32_t);                                          \
    extern "C" int V(cc_neuron_step)(const cc_shard*, void*);                               \
    extern "C" int V(cc_ingest)(const cc_shard*, const uint32_t*, const double*, const int32_t*, \
                                void*);                                                     \
    extern "C" int V(cc_pack_aer)(const cc_shard*, const uint32_t*, int32_t, int32_t, int64_t*, \
                                  const int32_t*, void*);                                   \
    extern "C" int V(cc_ingest_aer)(const cc_shard*, const int64_t*, int32_t, int32_t, void*); \
    extern "C" int V(cc_exchange_ingest)(const cc_shard*, void*);                           \
    extern "C" int V(cc_test_math)(int32_t, const double*, double*, int64_t, void*);
CC_DECL(A)
#if CC_NSUB_B != CC_NSUB_A
CC_DECL(B)
#endif

// which: 0 = variant A, 1 = variant B, -1 = not compiled in
static int variant_of(int32_t n_sub) {
    if (n_sub == CC_NSUB_A) return 0;
    if (n_sub == CC_NSUB_B) return 1;
    return -1;
}
static int bad_variant(const char* who, const cc_shard* sh) {
    if (!sh) return cc_set_error("%s: null shard", who);
    return cc_set_error("%s: cc_shard.n_sub = %d, this library carries %d and %d", who,
                        (int)sh->n_sub, CC_NSUB_A, CC_NSUB_B);
}
#if CC_NSUB_B != CC_NSUB_A
#define CC_DISPATCH(who, sh, call_a, call_b)                                   \
    switch ((sh) ? variant_of((sh)->n_sub) : -1) {                             \
        case 0: return call_a;                                                  \
        case 1: return call_b;                                                  \
        default: return bad_variant(who, sh);                                   \
    }
#else
#define CC_DISPATCH(who, sh, call_a, call_b)                                   \
    if ((sh) && variant_of((sh)->n_sub) == 0) return call_a;                   \
    return bad_variant(who, sh);
#endif

extern "C" int32_t cc_cnt_stride(int32_t n_sub) {
    return variant_of(n_sub) < 0 ? 0 : CC_CNT_STRIDE_FOR(n_sub);
}

extern "C" int cc_prepare(void) {
    if (const int rc = A(cc_prepare)()) return rc;
#if CC_NSUB_B != CC_NSUB_A
    if (const int rc = B(cc_prepare)()) return rc;
#endif
    return 0;
}

extern "C" int cc_deliver(const cc_shard* sh, void* stream) {
    CC_DISPATCH("cc_deliver", sh, A(cc_deliver)(sh, stream), B(cc_deliver)(sh, stream))
}

extern "C" int cc_neuron_step(const cc_shard* sh, void* stream) {
    CC_DISPATCH("cc_neuron_step", sh, A(cc_neuron_step)(sh, stream), B(cc_neuron_step)(sh, stream))
}

extern "C" int32_t cc_kernels_per_step(const cc_shard* sh) {
    if (!sh || variant_of(sh->n_sub) < 0) return 0;
    CC_DISPATCH("cc_kernels_per_step", sh, A(cc_kernels_per_step)(sh), B(cc_kernels_per_step)(sh))
}

extern "C" int32_t cc_stage_warps(const cc_shard* sh) {
    if (!sh || variant_of(sh->n_sub) < 0) return 0;
    CC_DISPATCH("cc_stage_warps", sh, A(cc_stage_warps)(sh->d_max), B(cc_stage_warps)(sh->d_max))
}

// Entry points that do not depend on the input lists: variant A's copies.
extern "C" int cc_build_dseg(const int64_t* row_off, const uint8_t* syn_d, int64_t n_rows,
                             int32_t d_max, int32_t stride, uint16_t* out, unsigned* err,
                             void* stream) {
    return A(cc_build_dseg)(row_off, syn_d, n_rows, d_max, stride, out, err, stream);
}
extern "C" int cc_init_state(const cc_shard* sh, void* stream) {
    return A(cc_init_state)(sh, stream);
}
extern "C" int cc_ingest(const cc_shard* sh, const uint32_t* in_gid, const double* in_t,
                         const int32_t* in_n, void* stream) {
    return A(cc_ingest)(sh, in_gid, in_t, in_n, stream);
}
extern "C" int cc_pack_aer(const cc_shard* sh, const uint32_t* dest_mask_by_local, int32_t n_dest,
                           int32_t cap, int64_t* send, const int32_t* local_of_col, void* stream) {
    return A(cc_pack_aer)(sh, dest_mask_by_local, n_dest, cap, send, local_of_col, stream);
}
extern "C" int cc_ingest_aer(const cc_shard* sh, const int64_t* recv, int32_t n_src, int32_t cap,
                             void* stream) {
    return A(cc_ingest_aer)(sh, recv, n_src, cap, stream);
}
extern "C" int cc_exchange_ingest(const cc_shard* sh, void* stream) {
    return A(cc_exchange_ingest)(sh, stream);
}
extern "C" int cc_test_math(int32_t kind, const double* x, double* out, int64_t n, void* stream) {
    return A(cc_test_math)(kind, x, out, n, stream);
}

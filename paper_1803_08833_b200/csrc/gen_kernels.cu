// Connectivity generator (north-star kernel 1), bit-exact with the reference.
//
// For every listed source neuron one warp replays the reference's per-source
// draws (connectivity.py:383-417) from the same Philox4x64-10 streams:
//   CONNECTIVITY  word j decides candidate j of the layout (u < p)
//   WEIGHT        the k-th selected synapse gets the k-th ziggurat normal
//   DELAY         the k-th selected synapse gets the k-th uniform (random
//                 access) or ziggurat exponential draw
// but keeps only the synapses whose target column this shard owns, so no
// construction exchange is needed (network.py:189-295 becomes local).
// Rows are written sorted by (delay, layout order) = the reference's stable
// lexsort by (source, delay) (network.py:257).
//
// Sequential ziggurat streams are walked warp-cooperatively: 32 lanes try the
// 99 % single-word fast path on consecutive words; the first lane that needs
// the slow path finishes its draw serially and the window restarts after it.
#include "cc_common.cuh"

namespace {

constexpr int GEN_BLOCK = 128;
constexpr int GEN_WARPS = GEN_BLOCK / 32;

struct SrcInfo {
    uint32_t gid;
    int col, self_local, nblk, last_owned;
    bool exc;
};

__device__ __forceinline__ SrcInfo src_info(const cc_gen& g, uint32_t gid) {
    SrcInfo s;
    s.gid = gid;
    s.col = (int)(gid / (uint32_t)g.n_col);
    s.self_local = (int)(gid % (uint32_t)g.n_col);
    s.exc = s.self_local < g.n_exc_col;
    s.nblk = s.exc ? g.blk_count[s.col] : 1;
    s.last_owned = -1;
    for (int b = 0; b < s.nblk; ++b)
        if (g.col_local[g.blk_col[(size_t)s.col * g.kmax + b]] >= 0) s.last_owned = b;
    return s;
}

// Selection bits of candidates [c0, c0 + 4) (one Philox block when aligned);
// bit i set when candidate c0+i exists (< c_end), is not the autapse slot and
// draws u < p of its block.
__device__ __forceinline__ unsigned sel4(const cc_gen& g, const SrcInfo& s, int64_t q,
                                         int64_t c_end) {
    const cc_philox_block pb = cc_philox4x64((uint64_t)q + 1, s.gid, 0, CC_DOMAIN, g.seed, 1);
    unsigned bits = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t j = q * 4 + i;
        if (j >= c_end) break;
        const int b = (int)(j / g.n_col);
        if (b == 0 && (int)j == s.self_local) continue;          // autapse slot, p = 0
        const double p = g.blk_p[(size_t)s.col * g.kmax + b];
        if (cc_u53(pb.v[i]) < p) bits |= 1u << i;
    }
    return bits;
}

// Per-block selected counts of blocks [0, last_owned] into cnt[] (shared).
__device__ void count_blocks(const cc_gen& g, const SrcInfo& s, int* cnt) {
    const int lane = threadIdx.x & 31;
    for (int b = lane; b <= s.last_owned; b += 32) cnt[b] = 0;
    __syncwarp();
    const int64_t c_end = (int64_t)(s.last_owned + 1) * g.n_col;
    const int64_t nq = (c_end + 3) / 4;
    for (int64_t q = lane; q < nq; q += 32) {
        const unsigned bits = sel4(g, s, q, c_end);
        if (!bits) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (bits >> i & 1u) atomicAdd(&cnt[(int)((q * 4 + i) / g.n_col)], 1);
    }
    __syncwarp();
}

// rank_base[b] = exclusive prefix of cnt; own_base[b] = prefix over owned blocks.
__device__ int scan_blocks(const cc_gen& g, const SrcInfo& s, const int* cnt, int* rank_base,
                           int* own_base) {
    const int lane = threadIdx.x & 31;
    int r = 0, o = 0;
    for (int b0 = 0; b0 <= s.last_owned; b0 += 32) {
        const int b = b0 + lane;
        int c = 0, oc = 0;
        if (b <= s.last_owned) {
            c = cnt[b];
            oc = g.col_local[g.blk_col[(size_t)s.col * g.kmax + b]] >= 0 ? c : 0;
        }
        int xc = c, xo = oc;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
            const int yc = __shfl_up_sync(0xffffffffu, xc, k);
            const int yo = __shfl_up_sync(0xffffffffu, xo, k);
            if (lane >= k) { xc += yc; xo += yo; }
        }
        if (b <= s.last_owned) { rank_base[b] = r + xc - c; own_base[b] = o + xo - oc; }
        r += __shfl_sync(0xffffffffu, xc, 31);
        o += __shfl_sync(0xffffffffu, xo, 31);
    }
    __syncwarp();
    if (lane == 0) { rank_base[s.last_owned + 1] = r; own_base[s.last_owned + 1] = o; }
    __syncwarp();
    return o;
}

__device__ __forceinline__ int block_of_rank(const int* rank_base, int nb, int r) {
    int lo = 0, hi = nb;                  // largest b with rank_base[b] <= r
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (rank_base[mid] <= r) lo = mid; else hi = mid;
    }
    return lo;
}

// Warp-cooperative walk over a sequential ziggurat stream: calls
// emit(rank, value) for ranks [0, r_end) in parallel batches.
template <bool NORMAL, typename Emit>
__device__ void zig_walk(uint64_t seed, uint64_t purpose, uint64_t gid, int r_end, Emit emit) {
    const int lane = threadIdx.x & 31;
    uint64_t pos = 0;
    int r = 0;
    while (r < r_end) {
        // fast path attempt on word pos + lane
        const uint64_t w = cc_philox_word(seed, purpose, gid, pos + lane);
        bool ok;
        double x;
        if (NORMAL) {
            const int idx = (int)(w & 0xff);
            const uint64_t rr = w >> 8;
            const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffull;
            x = (double)rabs * cc_zig_wi[idx];
            if (rr & 1) x = -x;
            ok = rabs < cc_zig_ki[idx];
        } else {
            const uint64_t ri = (w >> 3) >> 8;
            const int idx = (int)((w >> 3) & 0xff);
            x = (double)ri * cc_zig_we[idx];
            ok = ri < cc_zig_ke[idx];
        }
        const unsigned bad = __ballot_sync(0xffffffffu, !ok);
        const int f = bad ? __ffs(bad) - 1 : 32;
        if (lane < f && r + lane < r_end) emit(r + lane, x);
        if (f == 32) { pos += 32; r += 32; continue; }
        // lane f's draw takes the slow path: replay it serially
        double v = 0.0;
        uint64_t npos = 0;
        if (lane == 0) {
            cc_philox_stream st;
            st.init(seed, purpose, gid, pos + f);
            v = NORMAL ? cc_std_normal(st) : cc_std_exponential(st);
            npos = st.pos;
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        npos = __shfl_sync(0xffffffffu, npos, 0);
        if (lane == 0 && r + f < r_end) emit(r + f, v);
        pos = npos;
        r += f + 1;
    }
    __syncwarp();
}

struct Stage {               // per-warp staging of one source's owned synapses
    int32_t* tgt;            // global target gid
    float* w;
    uint8_t* d;
};

__device__ __forceinline__ uint64_t wire_mix(uint32_t src, uint32_t tgt, uint16_t d,
                                             uint16_t flags, float w) {
    const uint64_t lo = (uint64_t)src | ((uint64_t)tgt << 32);
    const uint64_t hi = (uint64_t)d | ((uint64_t)flags << 16)
                        | ((uint64_t)__float_as_uint(w) << 32);
    return cc_splitmix64(lo ^ cc_splitmix64(hi));
}

template <bool FILL>
__global__ void __launch_bounds__(GEN_BLOCK)
k_gen(const cc_gen g, const uint32_t* __restrict__ src_gid, int64_t n_src,
      int64_t* row_len, const int64_t* row_start, int32_t* syn_tgt, float* syn_w,
      uint8_t* syn_d, unsigned long long* checksum, float* scratch, int64_t scratch_per_warp,
      unsigned* err) {
    extern __shared__ int gsm[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int kpad = g.kmax + 1;
    int* cnt = gsm + warp * (3 * kpad + 256);
    int* rank_base = cnt + kpad;
    int* own_base = rank_base + kpad;
    int* dcur = own_base + kpad;
    const int64_t gw = ((int64_t)blockIdx.x * GEN_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * GEN_BLOCK) >> 5;
    Stage stg;
    if (FILL) {
        float* base = scratch + gw * scratch_per_warp;
        const int64_t cap = scratch_per_warp / 3;   // 3 words per staged synapse (d packed in 1)
        stg.tgt = reinterpret_cast<int32_t*>(base);
        stg.w = base + cap;
        stg.d = reinterpret_cast<uint8_t*>(base + 2 * cap);
    }
    unsigned long long csum = 0;
    for (int64_t i = gw; i < n_src; i += nw) {
        const SrcInfo s = src_info(g, src_gid[i]);
        if (s.last_owned < 0) {
            if (!FILL && lane == 0) row_len[i] = 0;
            continue;
        }
        count_blocks(g, s, cnt);
        const int n_own = scan_blocks(g, s, cnt, rank_base, own_base);
        if (!FILL) {
            if (lane == 0) row_len[i] = n_own;
            continue;
        }
        if (n_own == 0) continue;
        if ((int64_t)n_own * 3 > scratch_per_warp ||
            n_own != (int)(row_start[i + 1] - row_start[i])) {
            if (lane == 0) atomicOr(err, CC_ERR_GEN);
            continue;
        }
        // (1) targets of owned blocks, layout order
        for (int b = 0; b <= s.last_owned; ++b) {
            const int tcol = g.blk_col[(size_t)s.col * g.kmax + b];
            if (g.col_local[tcol] < 0 || cnt[b] == 0) continue;
            const int64_t c0 = (int64_t)b * g.n_col, c1 = c0 + g.n_col;
            int wpos = own_base[b];
            // lanes take consecutive 4-word Philox blocks covering [c0, c1)
            for (int64_t q0 = c0 / 4; q0 * 4 < c1; q0 += 32) {
                const int64_t q = q0 + lane;
                unsigned bits = 0;
                if (q * 4 < c1) {
                    bits = sel4(g, s, q, c1);
                    // drop candidates before c0 (previous block shares this Philox block)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (q * 4 + k < c0) bits &= ~(1u << k);
                }
                const int nb = __popc(bits);
                int x = nb;
#pragma unroll
                for (int k = 1; k < 32; k <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, k);
                    if (lane >= k) x += y;
                }
                int p = wpos + x - nb;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (bits >> k & 1u) {
                        const int64_t j = q * 4 + k;
                        stg.tgt[p++] = (int32_t)((int64_t)tcol * g.n_col + (j - c0));
                    }
                }
                wpos += __shfl_sync(0xffffffffu, x, 31);
            }
        }
        __syncwarp();
        const int nb_all = s.last_owned + 1;
        const int r_end = rank_base[nb_all];
        auto staged_index = [&](int r) -> int {
            const int b = block_of_rank(rank_base, nb_all, r);
            if (g.col_local[g.blk_col[(size_t)s.col * g.kmax + b]] < 0) return -1;
            return own_base[b] + (r - rank_base[b]);
        };
        // (2) weights: k-th normal of the WEIGHT stream for rank k (connectivity.py:403-409)
        zig_walk<true>(g.seed, 2, s.gid, r_end, [&](int r, double z) {
            const int si = staged_index(r);
            if (si < 0) return;
            const int tl = stg.tgt[si] % g.n_col;
            const bool texc = tl < g.n_exc_col;
            const double j = s.exc ? (texc ? g.j_ee : g.j_ei) : (texc ? g.j_ie : g.j_ii);
            double w = j * (1.0 + g.sd_frac * z);
            if (s.exc) { if (w < 0.0) w = 0.0; } else { if (w > 0.0) w = 0.0; }
            stg.w[si] = __double2float_rn(w);
        });
        // (3) delays (connectivity.py:410-416)
        auto put_delay = [&](int si, double d_ms) {
            double st = rint(d_ms / g.dt);
            long long k = (long long)st;
            k = k < 1 ? 1 : (k > g.d_max ? g.d_max : k);
            stg.d[si] = (uint8_t)k;
        };
        if (g.delay_kind == 0) {
            for (int b = 0; b < nb_all; ++b) {
                if (g.col_local[g.blk_col[(size_t)s.col * g.kmax + b]] < 0) continue;
                for (int k = lane; k < cnt[b]; k += 32) {
                    const int r = rank_base[b] + k;
                    const double u = cc_u53(cc_philox_word(g.seed, 3, s.gid, (uint64_t)r));
                    put_delay(own_base[b] + k, g.d_lo + g.d_scale * u);
                }
            }
        } else {
            zig_walk<false>(g.seed, 3, s.gid, r_end, [&](int r, double e) {
                const int si = staged_index(r);
                if (si >= 0) put_delay(si, g.d_scale * e);
            });
        }
        __syncwarp();
        // (4) stable counting sort by delay into the row
        for (int k = lane; k < 256; k += 32) dcur[k] = 0;
        __syncwarp();
        for (int si = lane; si < n_own; si += 32) atomicAdd(&dcur[stg.d[si]], 1);
        __syncwarp();
        if (lane == 0) {
            int acc = 0;
            for (int k = 0; k < 256; ++k) { const int c = dcur[k]; dcur[k] = acc; acc += c; }
        }
        __syncwarp();
        const int64_t r0 = row_start[i];
        const uint16_t flags = s.exc ? 1 : 0;
        for (int si0 = 0; si0 < n_own; si0 += 32) {
            const int si = si0 + lane;
            const bool v = si < n_own;
            const int d = v ? stg.d[si] : 256 + lane;      // unique dummy key when idle
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const int before = __popc(peers & ((1u << lane) - 1u));
            int pos = 0;
            if (v) pos = dcur[d] + before;
            __syncwarp();
            if (v && before == __popc(peers) - 1) dcur[d] += __popc(peers);
            __syncwarp();
            if (v) {
                const int32_t tg = stg.tgt[si];
                const float w = stg.w[si];
                const int tcol = tg / g.n_col;
                syn_tgt[r0 + pos] = g.col_local[tcol] * g.n_col + tg % g.n_col;
                syn_w[r0 + pos] = w;
                syn_d[r0 + pos] = (uint8_t)d;
                csum += wire_mix(s.gid, (uint32_t)tg, (uint16_t)d, flags, w);
            }
        }
        __syncwarp();
    }
    if (FILL) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
        if (lane == 0 && csum) atomicAdd(checksum, csum);
    }
}

// Wire-record checksum of existing rows (imported connectivity).
__global__ void k_csr_checksum(const int64_t* row_off, const uint32_t* src_gid, int64_t n_src,
                               const int32_t* tgt_global, const float* w, const uint8_t* d,
                               int n_col, int n_exc_col, unsigned long long* checksum) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long cs = 0;
    for (int64_t i = gw; i < n_src; i += nw) {
        const uint32_t src = src_gid[i];
        const uint16_t flags = ((int)(src % (uint32_t)n_col) < n_exc_col) ? 1 : 0;
        for (int64_t k = row_off[src] + lane; k < row_off[src + 1]; k += 32)
            cs += wire_mix(src, (uint32_t)tgt_global[k], d[k], flags, w[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
    if (lane == 0 && cs) atomicAdd(checksum, cs);
}

// Stream probes for the parity tests.
__global__ void k_test_philox(uint64_t seed, uint64_t purpose, uint64_t a, int64_t n, int kind,
                              double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    cc_philox_stream st;
    st.init(seed, purpose, a, 0);
    for (int64_t i = 0; i < n; ++i) {
        double v;
        switch (kind) {
            case 0: { const uint64_t w = st.next(); v = __longlong_as_double((long long)w); break; }
            case 1: v = st.next_double(); break;
            case 2: v = cc_std_normal(st); break;
            default: v = cc_std_exponential(st); break;
        }
        out[i] = v;
    }
}

// Warp-cooperative ziggurat walk probe (exercises zig_walk's batching).
__global__ void k_test_zig_walk(uint64_t seed, uint64_t purpose, uint64_t a, int n, int normal,
                                double* out) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    if (normal) zig_walk<true>(seed, purpose, a, n, [&](int r, double v) { out[r] = v; });
    else zig_walk<false>(seed, purpose, a, n, [&](int r, double v) { out[r] = v; });
}

__global__ void k_test_cu(uint64_t seed, uint64_t purpose, const uint64_t* a, uint64_t b,
                          const uint64_t* k, int64_t n, double* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t h = cc_splitmix64(seed ^ CC_DOMAIN);
    h = cc_splitmix64(h ^ purpose);
    h = cc_splitmix64(h ^ a[i]);
    h = cc_splitmix64(h ^ b);
    h = cc_splitmix64(h ^ k[i]);
    out[i] = cc_u53(h);
}

}  // namespace

extern "C" int cc_set_error(const char* fmt, ...);
extern "C" int cc_check_launch(const char* what);

static int gen_grid() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return (n > 0 ? n : 148) * 8;
}

static size_t gen_smem(const cc_gen* g) {
    return (size_t)GEN_WARPS * (3 * (g->kmax + 1) + 256) * sizeof(int);
}

static int gen_prep(const cc_gen* g) {
    const size_t sm = gen_smem(g);
    if (sm > 48 * 1024) {
        cudaFuncSetAttribute(k_gen<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_gen<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    }
    return 0;
}

extern "C" int cc_gen_count(const cc_gen* g, const uint32_t* src_gid, int64_t n_src,
                            int64_t* row_len, unsigned* err, void* stream) {
    if (!g) return cc_set_error("cc_gen_count: null spec");
    if (n_src == 0) return 0;
    gen_prep(g);
    k_gen<false><<<gen_grid(), GEN_BLOCK, gen_smem(g), (cudaStream_t)stream>>>(
        *g, src_gid, n_src, row_len, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, err);
    return cc_check_launch("k_gen<count>");
}

extern "C" int cc_gen_fill(const cc_gen* g, const uint32_t* src_gid, int64_t n_src,
                           const int64_t* row_start, int32_t* syn_tgt, float* syn_w,
                           uint8_t* syn_d, unsigned long long* checksum, float* scratch,
                           int64_t scratch_per_warp, unsigned* err, void* stream) {
    if (!g) return cc_set_error("cc_gen_fill: null spec");
    if (n_src == 0) return 0;
    gen_prep(g);
    k_gen<true><<<gen_grid(), GEN_BLOCK, gen_smem(g), (cudaStream_t)stream>>>(
        *g, src_gid, n_src, nullptr, row_start, syn_tgt, syn_w, syn_d, checksum, scratch,
        scratch_per_warp, err);
    return cc_check_launch("k_gen<fill>");
}

extern "C" int64_t cc_gen_warps(void) { return (int64_t)gen_grid() * GEN_WARPS; }

extern "C" int cc_csr_checksum(const int64_t* row_off, const uint32_t* src_gid, int64_t n_src,
                               const int32_t* syn_tgt_global, const float* syn_w,
                               const uint8_t* syn_d, int32_t n_col, int32_t n_exc_col,
                               unsigned long long* checksum, void* stream) {
    if (n_src == 0) return 0;
    k_csr_checksum<<<gen_grid(), 256, 0, (cudaStream_t)stream>>>(
        row_off, src_gid, n_src, syn_tgt_global, syn_w, syn_d, n_col, n_exc_col, checksum);
    return cc_check_launch("k_csr_checksum");
}

extern "C" int cc_test_philox(uint64_t seed, uint64_t purpose, uint64_t a, int64_t n,
                              int32_t kind, double* out, void* stream) {
    if (kind >= 10) {
        k_test_zig_walk<<<1, 32, 0, (cudaStream_t)stream>>>(seed, purpose, a, (int)n,
                                                            kind == 12 ? 1 : 0, out);
        return cc_check_launch("k_test_zig_walk");
    }
    k_test_philox<<<1, 1, 0, (cudaStream_t)stream>>>(seed, purpose, a, n, kind, out);
    return cc_check_launch("k_test_philox");
}

extern "C" int cc_test_counter_uniforms(uint64_t seed, uint64_t purpose, const uint64_t* a,
                                        uint64_t b, const uint64_t* k, int64_t n, double* out,
                                        void* stream) {
    if (n == 0) return 0;
    k_test_cu<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(seed, purpose, a, b, k,
                                                                        n, out);
    return cc_check_launch("k_test_cu");
}

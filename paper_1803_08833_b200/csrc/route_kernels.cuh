// Routed delivery (included by sim_kernels.cu inside its anonymous namespace,
// after k_deliver): the expand/arborize + DelayRing.insert/drain step of the
// reference (engine.py:338-367, :124-163) in two passes for high event
// volumes.
//
// k_deliver deposits every event with one scattered 8 B store into one of
// n_groups x n_sub input lists; on the exponential grids (a row's targets
// spread one per list) those stores are the kernel's cost (measured with the
// probe build at the 31 Hz stress point of config 2: 1181 us per step, 441 us
// without the record stores, 215 us for the loads alone).  Here no event is
// stored on its own: each pass sorts a tile of events by destination in
// shared memory and copies whole runs.
//
//   k_route  pass 1.  A block stages up to RT_NB arriving events (the same
//            units, descriptors and CSR loads as k_deliver), counting-sorts
//            them by region of 2^l1_rb consecutive target neurons, reserves
//            each region's run with one atomic and copies the runs out:
//            10 B per event (spike_ref, weight bits, target within region).
//   k_bin    pass 2.  A block takes a tile of BN_T records of one region,
//            counting-sorts them by input list (group x sub-list), reserves
//            each list's run with one atomic on the list's fill counter - the
//            same counter k_deliver and k_stage's tail use, so all depositors
//            compose - and copies the runs out as the usual 8 B records.
//
// The input lists end up holding the same multiset of records as with
// k_deliver (the readers order a neuron's inputs by (time, source, weight)
// themselves), so rasters stay bit-identical.

// (the checked test variant is built with one record per thread and three
// k_route blocks, so that the small golden cases run through many tiles)
#ifndef CC_RT_PER_THREAD
#define CC_RT_PER_THREAD 12
#endif
#ifndef CC_BN_PER_THREAD
#define CC_BN_PER_THREAD 8
#endif
#ifndef CC_RT_BLOCKS
#define CC_RT_BLOCKS 0       // k_route blocks (0: one per SM)
#endif
#ifndef CC_RT_THREADS
#define CC_RT_THREADS 1024
#endif
#ifndef CC_RT_MINB
#define CC_RT_MINB 1
#endif
#ifndef CC_BN_MINB
#define CC_BN_MINB 2
#endif
constexpr int RT_THREADS = CC_RT_THREADS;
constexpr int RT_RPT = CC_L1_MAX_REGIONS / RT_THREADS;   // regions scanned per thread
constexpr int RT_PER_THREAD = CC_RT_PER_THREAD;
constexpr int RT_NB = RT_THREADS * RT_PER_THREAD;     // events staged per tile
static_assert(RT_NB < 65536, "tile positions are stored in 16 bits");
static_assert(CC_L1_MAX_REGIONS == RT_RPT * RT_THREADS, "k_route scans whole regions per thread");

constexpr size_t route_smem_bytes() {
    return (size_t)RT_NB * (4 + 4 + 4 + 2) + (size_t)CC_L1_MAX_REGIONS * 4 * 3;
}

// Exclusive block scan of one value per thread (blockDim.x a multiple of 32,
// <= 1024); wsum: 33 words of shared memory.  Two barriers.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* wsum, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
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
        wsum[lane] = w;                     // inclusive over warps (>= nwarp: the total)
    }
    __syncthreads();
    total = wsum[31];
    return (warp ? wsum[warp - 1] : 0u) + x - v;
}

__global__ void __launch_bounds__(RT_THREADS, CC_RT_MINB)
k_route(const cc_shard sh) {
    cc_ctl* ctl = sh.ctl;
    const long long t = *(volatile long long*)&ctl->t;
    if (*(volatile unsigned*)&ctl->error_bits) return;      // failed run: stop working
    const int L = sh.log_slots, D = sh.d_max;
    __shared__ unsigned s_n[DEL_DMAX], s_pre[DEL_DMAX + 1];
    __shared__ unsigned s_c0, s_fill, s_end, s_claim;
    __shared__ uint32_t s_wsum[33];
    __shared__ unsigned long long blk_ev;
    extern __shared__ __align__(16) unsigned char rt_smem[];
    uint32_t* s_ref = reinterpret_cast<uint32_t*>(rt_smem);
    uint32_t* s_w = s_ref + RT_NB;
    uint32_t* s_tgt = s_w + RT_NB;
    uint32_t* s_hist = s_tgt + RT_NB;
    uint32_t* s_start = s_hist + CC_L1_MAX_REGIONS;
    uint32_t* s_gbase = s_start + CC_L1_MAX_REGIONS;
    uint16_t* s_pos = reinterpret_cast<uint16_t*>(s_gbase + CC_L1_MAX_REGIONS);
    if (blockIdx.x == 0 && threadIdx.x == 0) deliver_prologue(sh, t);
    if (threadIdx.x == 32) s_c0 = *(volatile unsigned*)&sh.tailc[0];
    if (threadIdx.x == 64) { s_fill = 0u; s_end = 0xffffffffu; s_claim = 0u; blk_ev = 0ull; }
    for (int r = threadIdx.x; r < CC_L1_MAX_REGIONS; r += RT_THREADS) s_hist[r] = 0u;
    const int t_mod = (int)pos_mod(t, L);
    unit_prefix(sh, t_mod, D, s_n, s_pre);                   // (barriers)
    const unsigned n_units = s_pre[D];
    const unsigned c0 = min(s_c0, s_pre[D - 1]);
    const int lane = threadIdx.x & 31;
    constexpr int U = CC_DEL_U;
    const int lps = del_lps(sh);
    const int SPAN = lps * U;                                // synapses per spike per pass
    const int sl = lane & (lps - 1);
    const bool cnt_lane = sl == 0;                           // one lane per spike counts
    const unsigned lt_mask = (1u << lane) - 1u;
    const int RB = sh.l1_rb;
    const int n_reg = sh.n_regions;
    const uint32_t rmask = (1u << RB) - 1u;
    const size_t cap = (size_t)sh.l1_cap;
    uint32_t* gcnt = sh.l1_cnt + (size_t)(t & 1) * n_reg * CC_L1_STRIDE;
    unsigned long long my_ev = 0ull;
    int kc = 0, p = 0;
    uint64_t st = 0;
    uint32_t ln = 0, rf = 0, lmax = 0;
    bool have = false, done = false;
    for (;;) {
        // ---- fill: warps claim units and stage their passes until the tile is full
        while (!done) {
            if (!have) {
                unsigned c = 0;
                if (lane == 0) c = atomicAdd(&s_claim, 1u);
                c = __shfl_sync(0xffffffffu, c, 0);
                const unsigned long long uu = (unsigned long long)c0 + blockIdx.x +
                                              (unsigned long long)c * gridDim.x;
                if (uu >= n_units) { done = true; break; }
                unit_desc(sh, t_mod, s_n, s_pre, (unsigned)uu, kc, st, ln, rf);
                lmax = warp_max_u32(ln);
                p = 0;
                if (cnt_lane) my_ev += ln;
                if (lmax == 0) continue;
                have = true;
            }
            // staging slots of this pass: lane-major within each k (conflict-free)
            unsigned pre[U + 1];
            pre[0] = 0u;
            unsigned mine[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const bool v = (uint32_t)((p * U + k) * lps + sl) < ln;
                const unsigned b = __ballot_sync(0xffffffffu, v);
                mine[k] = pre[k] + __popc(b & lt_mask);
                pre[k + 1] = pre[k] + __popc(b);
            }
            const unsigned total = pre[U];
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&s_fill, total);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base + total > (unsigned)RT_NB) {
                // tile full: keep the pass.  The cursor stays past the end, so
                // every later reservation fails too and the staged events are
                // exactly [0, first failing base)
                if (lane == 0) atomicMin(&s_end, base);
                break;
            }
            int tg[U];
            float w[U];
            load_pass<U>(sh, st, ln, p, tg, w);
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (tg[k] < 0) continue;
                const unsigned i = base + mine[k];
                const unsigned reg = (unsigned)tg[k] >> RB;
                CC_CHK(ctl, i < (unsigned)RT_NB && reg < (unsigned)n_reg);
                s_ref[i] = rf;
                s_w[i] = __float_as_uint(w[k]);
                s_tgt[i] = (uint32_t)tg[k];
                s_pos[i] = (uint16_t)atomicAdd(&s_hist[reg], 1u);   // rank within (tile, region)
            }
            ++p;
            if ((uint32_t)(p * SPAN) >= lmax) have = false;
        }
        const int more = __syncthreads_or(!done);
        const unsigned n_ev = min(s_fill, s_end);
        // ---- region runs: scan the histogram, reserve each run in its region's array
        {
            uint32_t h[RT_RPT], sum = 0;
#pragma unroll
            for (int q = 0; q < RT_RPT; ++q) {
                const int r = RT_RPT * threadIdx.x + q;
                h[q] = s_hist[r];
                s_hist[r] = 0u;
                sum += h[q];
            }
            uint32_t tot;
            uint32_t ex = block_excl_scan(sum, s_wsum, tot);             // (barriers)
            CC_CHK(ctl, tot == n_ev);
#pragma unroll
            for (int q = 0; q < RT_RPT; ++q) {
                const int r = RT_RPT * threadIdx.x + q;
                s_start[r] = ex;
                ex += h[q];
                if (h[q]) {
                    const uint32_t g = atomicAdd(&gcnt[(size_t)r * CC_L1_STRIDE], h[q]);
                    s_gbase[r] = g;
                    if ((size_t)g + h[q] > cap) cc_raise(ctl, CC_ERR_OVERFLOW_BIN, t);
                }
            }
        }
        __syncthreads();
        // ---- sorted position of every staged event, then the permutation
        uint16_t pos[RT_PER_THREAD];
#pragma unroll
        for (int k = 0; k < RT_PER_THREAD; ++k) {
            const unsigned i = threadIdx.x + k * RT_THREADS;
            pos[k] = 0;
            if (i < n_ev) pos[k] = (uint16_t)(s_start[s_tgt[i] >> RB] + s_pos[i]);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < RT_PER_THREAD; ++k) {
            const unsigned i = threadIdx.x + k * RT_THREADS;
            if (i < n_ev) s_pos[pos[k]] = (uint16_t)i;
        }
        if (threadIdx.x == 0) { s_fill = 0u; s_end = 0xffffffffu; }
        __syncthreads();
        // ---- copy the runs out: consecutive threads, consecutive records of a run
#pragma unroll 4
        for (int k = 0; k < RT_PER_THREAD; ++k) {
            const unsigned j = threadIdx.x + k * RT_THREADS;
            if (j >= n_ev) break;
            const unsigned i = s_pos[j];
            const uint32_t tg = s_tgt[i];
            const unsigned reg = tg >> RB;
            const size_t d = (size_t)s_gbase[reg] + (j - s_start[reg]);
            if (d < cap) {
                const size_t o = (size_t)reg * cap + d;
                sh.l1_ref[o] = s_ref[i];
                sh.l1_w[o] = s_w[i];
                sh.l1_tgt[o] = (uint16_t)(tg & rmask);
            }
        }
        __syncthreads();
        if (!more) break;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_ev += __shfl_xor_sync(0xffffffffu, my_ev, o);
    if (lane == 0 && my_ev) atomicAdd(&blk_ev, my_ev);
    __syncthreads();
    if (threadIdx.x == 0 && blk_ev) atomicAdd(&ctl->del_events, blk_ev);
}

#ifndef CC_BN_THREADS
#define CC_BN_THREADS 512
#endif
constexpr int BN_THREADS = CC_BN_THREADS;
constexpr int BN_LPT = CC_L1_MAX_LISTS / BN_THREADS;      // lists scanned per thread
constexpr int BN_RPT = CC_L1_MAX_REGIONS / BN_THREADS;    // regions scanned per thread
constexpr int BN_PER_THREAD = CC_BN_PER_THREAD;
constexpr int BN_T = BN_THREADS * BN_PER_THREAD;       // records per tile
static_assert(CC_L1_MAX_LISTS == BN_LPT * BN_THREADS && CC_L1_MAX_REGIONS == BN_RPT * BN_THREADS,
              "k_bin scans whole lists / regions per thread");

// (ncnt_rb: log2 of the per-neuron counters behind the tile arrays, -1: none)
constexpr size_t bin_smem_bytes(int ncnt_rb = -1) {
    return (size_t)BN_T * (8 + 2) + (size_t)CC_L1_MAX_LISTS * 4 * 3 +
           ((size_t)(CC_L1_MAX_REGIONS + 1) * 4 + 15) / 16 * 16 +
           (ncnt_rb >= 0 ? ((size_t)4 << ncnt_rb) : 0);
}
// Per-neuron counts: CC_BN_TEAM blocks share a contiguous range of tiles (one
// region after the other), so that a block meets few regions and can keep its
// counts in shared memory, while the blocks running at a time still touch
// few regions' lists (fully contiguous ranges - a team of 1 - put 296 regions'
// lists in flight: k_bin +49 us at the stress point of config 2).
#ifndef CC_BN_TEAM
#define CC_BN_TEAM 4
#endif

__global__ void __launch_bounds__(BN_THREADS, CC_BN_MINB)
k_bin(const cc_shard sh) {
    cc_ctl* ctl = sh.ctl;
    const long long t = *(volatile long long*)&ctl->t;
    if (*(volatile unsigned*)&ctl->error_bits) return;      // failed run: stop working
    extern __shared__ __align__(16) unsigned char bn_smem[];
    uint64_t* s_rec = reinterpret_cast<uint64_t*>(bn_smem);
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_rec + BN_T);
    uint32_t* s_start = s_hist + CC_L1_MAX_LISTS;
    uint32_t* s_base = s_start + CC_L1_MAX_LISTS;
    uint32_t* s_tpre = s_base + CC_L1_MAX_LISTS;             // [n_regions + 1] tile prefix
    uint32_t* s_ncnt = s_tpre + (CC_L1_MAX_REGIONS + 1 + 3) / 4 * 4;   // [2^RB] if sh.l1_ncnt
    const bool count_n = sh.l1_ncnt != nullptr;
    uint16_t* s_list = reinterpret_cast<uint16_t*>(s_ncnt + (count_n ? (1 << sh.l1_rb) : 0));
    __shared__ uint32_t s_wsum[33];
    const int RB = sh.l1_rb;
    const int n_reg = sh.n_regions;
    const size_t cap = (size_t)sh.l1_cap;
    const uint32_t* gcnt = sh.l1_cnt + (size_t)(t & 1) * n_reg * CC_L1_STRIDE;
    const ListSet S = list_set(sh, t);
    const int K = sh.bin_cap;
    const size_t KS = (size_t)K + sh.bin_pad;
    [[maybe_unused]] const int nl = NSUB << (RB - 5);        // lists per region
    // tiles per region (every block computes the same prefix)
    uint32_t total_tiles;
    {
        uint32_t n4[BN_RPT], sum = 0;
#pragma unroll
        for (int q = 0; q < BN_RPT; ++q) {
            const int r = BN_RPT * threadIdx.x + q;
            uint32_t c = r < n_reg ? gcnt[(size_t)r * CC_L1_STRIDE] : 0u;
            c = (uint32_t)min((size_t)c, cap);
            n4[q] = (c + BN_T - 1) / BN_T;
            sum += n4[q];
        }
        uint32_t ex = block_excl_scan(sum, s_wsum, total_tiles);         // (barriers)
#pragma unroll
        for (int q = 0; q < BN_RPT; ++q) {
            s_tpre[BN_RPT * threadIdx.x + q] = ex;
            ex += n4[q];
        }
        if (threadIdx.x == BN_THREADS - 1) s_tpre[CC_L1_MAX_REGIONS] = ex;
    }
    // the other parity's region counters, for k_route(t + 1)
    if (blockIdx.x == 0) {
        uint32_t* other = sh.l1_cnt + (size_t)((t + 1) & 1) * n_reg * CC_L1_STRIDE;
        for (int r = threadIdx.x; r < n_reg; r += BN_THREADS) other[(size_t)r * CC_L1_STRIDE] = 0u;
    }
    for (int l = threadIdx.x; l < CC_L1_MAX_LISTS; l += BN_THREADS) s_hist[l] = 0u;
    if (count_n)
        for (int n = threadIdx.x; n < (1 << RB); n += BN_THREADS) s_ncnt[n] = 0u;
    __syncthreads();
    // per-neuron counts (sh.l1_ncnt): the block accumulates the records it
    // stores per neuron in shared memory and adds them to the global counts
    // when it leaves a region; its team's tiles are a contiguous range, dealt
    // round-robin inside the team.  Without the counts the tiles are dealt
    // round-robin over the whole grid.
    uint32_t* ncnt = count_n ? sh.l1_ncnt + (size_t)(t & 1) * sh.n_groups * 32 : nullptr;
    auto flush_counts = [&](int reg) {           // block-wide; barriers by the caller
        const size_t base = (size_t)reg << RB;
        for (int n = threadIdx.x; n < (1 << RB); n += BN_THREADS) {
            const uint32_t c = s_ncnt[n];
            if (c) {
                CC_CHK(ctl, base + n < (size_t)sh.n_groups * 32);
                atomicAdd(&ncnt[base + n], c);
                s_ncnt[n] = 0u;
            }
        }
    };
    uint32_t it_first = blockIdx.x, it_end = total_tiles, it_step = gridDim.x;
    if (count_n) {
        const unsigned team = min((unsigned)CC_BN_TEAM, gridDim.x);
        const unsigned n_teams = gridDim.x / team;             // (blocks past the last full team idle)
        const unsigned g = blockIdx.x / team, m = blockIdx.x % team;
        if (g < n_teams) {
            it_first = (uint32_t)((unsigned long long)total_tiles * g / n_teams) + m;
            it_end = (uint32_t)((unsigned long long)total_tiles * (g + 1) / n_teams);
        } else {
            it_first = it_end = 0u;
        }
        it_step = team;
    }
    int cur_reg = -1;
    for (uint32_t it = it_first; it < it_end; it += it_step) {
        // region of tile `it`: last r with s_tpre[r] <= it
        int lo = 0, hi = CC_L1_MAX_REGIONS;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_tpre[mid] <= it) lo = mid; else hi = mid;
        }
        const int reg = lo;
        CC_CHK(ctl, reg < n_reg && s_tpre[reg] <= it && it < s_tpre[reg + 1]);
        if (count_n && reg != cur_reg) {
            if (cur_reg >= 0) { flush_counts(cur_reg); __syncthreads(); }
            cur_reg = reg;
        }
        const uint32_t n_r = (uint32_t)min((size_t)gcnt[(size_t)reg * CC_L1_STRIDE], cap);
        const uint32_t j0 = (it - s_tpre[reg]) * BN_T;
        const uint32_t n_t = min((uint32_t)BN_T, n_r - j0);
        const size_t o0 = (size_t)reg * cap + j0;
        const unsigned list0 = ((unsigned)reg << (RB - 5)) * NSUB;
        uint32_t ref[BN_PER_THREAD], wb[BN_PER_THREAD];
        uint32_t tg[BN_PER_THREAD];                           // target | rank << 16
#pragma unroll
        for (int k = 0; k < BN_PER_THREAD; ++k) {
            const uint32_t j = threadIdx.x + k * BN_THREADS;
            if (j < n_t) {
                ref[k] = __ldg(sh.l1_ref + o0 + j);
                wb[k] = __ldg(sh.l1_w + o0 + j);
                tg[k] = __ldg(sh.l1_tgt + o0 + j);
            }
        }
#pragma unroll
        for (int k = 0; k < BN_PER_THREAD; ++k) {
            const uint32_t j = threadIdx.x + k * BN_THREADS;
            if (j < n_t) {
                const unsigned l = list_of((int)tg[k], 0);
                CC_CHK(ctl, l < (unsigned)nl);
                // (per-neuron counts: every record here, overflowed ones taken back below)
                if (count_n) atomicAdd(&s_ncnt[tg[k]], 1u);
                tg[k] |= atomicAdd(&s_hist[l], 1u) << 16;
            }
        }
        __syncthreads();
        {
            uint32_t h[BN_LPT], sum = 0;
#pragma unroll
            for (int q = 0; q < BN_LPT; ++q) {
                const int l = BN_LPT * threadIdx.x + q;
                h[q] = s_hist[l];
                s_hist[l] = 0u;
                sum += h[q];
            }
            uint32_t tot;
            uint32_t ex = block_excl_scan(sum, s_wsum, tot);             // (barriers)
            CC_CHK(ctl, tot == n_t);
#pragma unroll
            for (int q = 0; q < BN_LPT; ++q) {
                const int l = BN_LPT * threadIdx.x + q;
                s_start[l] = ex;
                ex += h[q];
                if (h[q]) s_base[l] = atomicAdd(&S.cnt[(size_t)(list0 + l) * CC_CNT_STRIDE], h[q]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BN_PER_THREAD; ++k) {
            const uint32_t j = threadIdx.x + k * BN_THREADS;
            if (j < n_t) {
                const unsigned l = list_of((int)(tg[k] & 0xffffu), 0);
                const uint32_t q = s_start[l] + (tg[k] >> 16);
                s_rec[q] = (uint64_t)((ref[k] << 5) | (tg[k] & 31u)) |
                           ((uint64_t)wb[k] << 32);
                s_list[q] = (uint16_t)l;
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < BN_PER_THREAD; ++k) {
            const uint32_t j = threadIdx.x + k * BN_THREADS;
            if (j >= n_t) break;
            const unsigned l = s_list[j];
            const uint32_t pos = s_base[l] + (j - s_start[l]);
            const uint64_t rec = s_rec[j];
            if (pos < (uint32_t)K) {
                S.rec[(size_t)(list0 + l) * KS + pos] = rec;
            } else {                                          // full list: the set's overflow list
                // (not a list record: taken back from its neuron's count -
                // the list's group and the record's lane)
                if (count_n) atomicSub(&s_ncnt[((l / NSUB) << 5) | ((uint32_t)rec & 31u)], 1u);
                const unsigned o = atomicAdd(S.ovf_cnt, 1u);
                atomicAdd(&ctl->ovf_total, 1ull);
                const uint32_t lo32 = (uint32_t)rec;
                // group of the record: sub-lists split a group's 32 lanes evenly
                const unsigned grp = (list0 + l) / NSUB;
                if (o < (unsigned)sh.ovf_cap)
                    S.ovf[o] = make_uint4(grp, lo32 & 31u, lo32 >> 5, (uint32_t)(rec >> 32));
                else cc_raise(ctl, CC_ERR_OVERFLOW_BIN, t);
            }
        }
        __syncthreads();
    }
    if (count_n && cur_reg >= 0) flush_counts(cur_reg);
    deliver_epilogue(sh, S, 0ull);
}

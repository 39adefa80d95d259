/*
 * corticarc_b200.h - C ABI of the B200 engine for the per-millisecond loop of
 * the DPSNN cortical simulator (arXiv 1803.08833; reference package
 * `corticarc`, /root/reference/pkg/src/corticarc).
 *
 * Plain pointers and sizes only: every device buffer is owned by the caller
 * (torch tensors in the Python host layer) and described to the library by a
 * `cc_shard` value.  All launchers are asynchronous on the given stream,
 * return 0 on success and a negative code on failure, with the message in
 * cc_last_error() (thread-local).
 *
 * Each entry point replaces a piece of the reference's hot path; the
 * reference interface it stands in for is cited per function.
 */
#ifndef CORTICARC_B200_H
#define CORTICARC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_ABI_VERSION 29

/* Input sub-lists per 32-neuron group, by target lane range: sub-list j of a
 * group holds the events of its lanes [32 j / n, 32 (j + 1) / n).  The library
 * carries the step kernels in two variants, CC_NSUB_A (one list per group:
 * fewest reservation atomics, best where a group's inputs fit two or three work
 * items) and CC_NSUB_B (a work item reads only the sub-lists of its own lanes:
 * best at high rates, where a group takes ten and more work items);
 * cc_shard.n_sub selects one per shard.  CC_CNT_STRIDE_FOR(n): u32 words between
 * the fill counters of consecutive lists (the host sizes bin_cnt with it). */
#ifndef CC_NSUB_A
#define CC_NSUB_A 1
#endif
#ifndef CC_NSUB_B
#define CC_NSUB_B 8
#endif
#define CC_CNT_STRIDE_FOR(n) ((n) >= 8 ? 8 : (n) >= 4 ? 16 : (n) >= 2 ? 32 : 64)
/* Work items are queued in this many size classes, largest first. */
#define CC_ITEM_CLASSES 8
/* Routed (two-pass) delivery, cc_shard.l1_cnt != NULL: regions of 2^l1_rb
 * consecutive neurons; at most CC_L1_MAX_REGIONS regions per shard and
 * CC_L1_MAX_LISTS input lists per region; region fill counters CC_L1_STRIDE
 * u32 words apart. */
#define CC_L1_MAX_REGIONS 2048
#define CC_L1_MAX_LISTS 1024
#define CC_L1_STRIDE 32
#define CC_L1_NCNT_MAX_RB 12

/* cc_shard.flags: measurement / test modes.  NO_TAIL_DELIVERY: k_stage's idle
 * warps do not deliver the next step's delay >= 2 events, so cc_deliver
 * deposits every arrival (bench.py's delivery roofline); PLAN_SEPARATE /
 * PLAN_FUSED force the planning pass into its own kernel / into k_stage
 * (tests; by default it is chosen by shard size).  Bits 32 / 256 / 512 / 1024
 * / 2048 are timing probes of builds with -DCC_TIMING_PROBES=1 (tools/). */
#define CC_FLAG_NO_TAIL_DELIVERY 0x1000
#define CC_FLAG_PLAN_SEPARATE    0x4000
#define CC_FLAG_PLAN_FUSED       0x8000

/* error bits raised by kernels into cc_ctl.error_bits */
#define CC_ERR_SPIKE_LOG      0x01u  /* more spikes in one step than log capacity   */
#define CC_ERR_DSEG           0x02u  /* CSR row longer than 65535 (delay segments)  */
#define CC_ERR_OVERFLOW_BIN   0x04u  /* overflow record list full                   */
#define CC_ERR_SCRATCH        0x08u  /* event staging scratch exhausted             */
#define CC_ERR_POISSON        0x10u  /* Poisson draw budget exceeded (engine.py:187)*/
#define CC_ERR_RASTER         0x20u  /* raster buffer full                          */
#define CC_ERR_OUTLIST        0x40u  /* exchange out-list full                      */
#define CC_ERR_GEN            0x80u  /* generator: row larger than planned          */
#define CC_ERR_EVREC          0x100u /* ordered-input record buffer full (one step) */
#define CC_ERR_GRIDSYNC       0x200u /* k_stage grid barrier timed out              */
#define CC_ERR_XWAIT          0x400u /* peer exchange: a source's step flag did not arrive in time */
#define CC_ERR_XCAP           0x800u /* peer exchange: destination region full     */
#define CC_ERR_CHECK          0x1000u/* checked build (CC_CHECKS): a bounds / protocol assertion
                                        failed; error_step holds its source line    */

/* Constants of one neuron population (model.py:44-86, NeuronBlock
 * per-neuron arrays model.py:243-267).  k1 = tau_c - tau_m and
 * k2 = tau_m * tau_c are pre-evaluated in float64 on the host (identical IEEE
 * results to the reference's in-line expressions, model.py:133); r_* are the
 * correctly rounded reciprocals 1/tau_m, 1/tau_c, 1/k2 used by the kernels'
 * exact division by these constants. */
typedef struct cc_pop {
    double tau_m, tau_c, E, V_theta, V_r, tau_arp, alpha_c, sfa, k1, k2;
    double r_tau_m, r_tau_c, r_k2;
} cc_pop;

/* Device-resident loop control and counters (one per shard). */
typedef struct cc_ctl {
    long long t;                          /* current step                     */
    unsigned long long rec_events;        /* expanded recurrent events        */
    unsigned long long ext_events;        /* generated external events        */
    unsigned long long n_spikes;
    unsigned long long raster_n;          /* entries in the raster buffer     */
    unsigned int pad2;
    unsigned int error_bits;
    long long error_step;
    unsigned int max_bin;                 /* max recurrent inputs of one neuron-step */
    unsigned int max_events;              /* max events of one neuron-step    */
    unsigned long long scratch_used;      /* staging events spilled (this step) */
    unsigned int out_n;                   /* exchange out-list fill           */
    unsigned int pad0;
    unsigned long long spilled_total;     /* neuron-steps that spilled smem   */
    unsigned long long ovf_total;         /* records that went to overflow    */
    unsigned int done_deliver;            /* last-block detection (deliver k.) */
    unsigned int ovf_grouped;             /* records grouped for this step    */
    unsigned long long stream_used;       /* event records used this step      */
    unsigned int done_stage;              /* last-block detection (stage k.)  */
    unsigned int n_rounds;                /* staging work items planned this step */
    unsigned int round_next;              /* next work item to claim          */
    unsigned int pad1;
    unsigned int cls_n[CC_ITEM_CLASSES];  /* work items queued per size class  */
    unsigned long long del_events;        /* recurrent events deposited by cc_deliver */
    unsigned long long tail_events;       /* ... by cc_neuron_step's idle warps (next step) */
    unsigned long long x_sent;            /* AER records pushed to peer shards */
    unsigned long long x_recv;            /* AER records received (all sources) */
} cc_ctl;

/* Peer exchange over NVLink (one process per GPU of one node; DESIGN.md
 * section 6).  Every rank owns one receive window (cudaMalloc'd by
 * cc_xwin_alloc, mapped into the other ranks with CUDA IPC) holding, per step
 * parity and per source rank, a region of AER records {gid, t lo, t hi, 0}
 * (uint4) and one flag word ((step + 1) << 32 | record count).  An entry
 * describes one such region: on the send side (xdst[d]) the region of THIS
 * rank in rank d's window, as mapped here; on the receive side (xsrc[s]) the
 * region of rank s in this rank's own window.  cap is the exact worst case:
 * the neurons of the source that have >= 1 synapse on the destination. */
typedef struct cc_xpeer {
    uint64_t rec[2];        /* region base (uint4 records) per step parity; 0 = no link */
    uint64_t flag[2];       /* flag word per step parity                         */
    uint32_t cap;           /* records per region                               */
    uint32_t pad;
} cc_xpeer;

/* One shard's device state.  Layout documented in DESIGN.md section 3. */
typedef struct cc_shard {
    /* sizes and constants */
    int32_t n_local;        /* neurons owned                                   */
    int32_t n_col;          /* neurons per column                              */
    int32_t n_exc_col;      /* excitatory slots per column                     */
    int32_t d_max;          /* SimConfig.d_max (delays 1..d_max steps)          */
    int32_t bin_cap;        /* records per input sub-list (per group and step)  */
    int32_t log_slots;      /* d_max + 1                                       */
    int32_t spk_cap;        /* spike-log entries per step (a power of two)     */
    int32_t seg_stride;     /* u16 per delay-segment table row: >= d_max + 1, %8 == 0 */
    int64_t ovf_cap;        /* overflow records per step                       */
    int64_t pad64_;
    int64_t raster_cap;     /* raster entries                                  */
    int64_t scratch_cap;    /* staging events (global spill, 56 B each)        */
    int64_t n_rows;         /* CSR rows (= global neuron count)                */
    int32_t out_cap;        /* exchange out-list capacity                      */
    int32_t ext_budget;     /* m = ceil(lam + 12 sqrt(lam)) + 20; 0 = no drive */
    int32_t n_probe;
    int32_t direct_log;     /* 1: neuron kernel logs its spikes itself (0: out-list only) */
    int32_t flags;          /* CC_FLAG_* mode bits (0 in production runs)       */
    int32_t plan_in_stage;  /* set by cc_neuron_step: k_stage runs the planning itself */
    int32_t del_lps_log2;   /* delivery: log2 lanes per spike (3: 4 spikes per warp unit, 4: 2) */
    int32_t n_sub;          /* input sub-lists per group: CC_NSUB_A or CC_NSUB_B        */
    uint64_t h2_ext;        /* splitmix chain prefix for EXTERNAL (rng.py:85-86)      */
    uint64_t h2_time;       /* ... for EXTERNAL_TIME                                  */
    uint64_t h2_init;       /* ... for INIT_STATE                                     */
    double dt;
    double ext_weight;      /* float64 external weight (engine.py:377-378)     */
    double ext_thresh;      /* exp(-lambda) evaluated with math.exp (engine.py:185) */
    cc_pop pop[2];          /* 0 excitatory, 1 inhibitory                      */

    /* neuron identity and state */
    const uint32_t* gid;    /* [n_local] global id                             */
    double* state;          /* [n_local][4] V, c, last_t, refr_until           */

    /* incoming-synapse CSR, rows keyed by global source id (network.py:114-152) */
    const int64_t* row_off; /* [n_rows + 1]                                    */
    const int32_t* syn_tgt; /* [S] local target index                          */
    const float* syn_w;     /* [S] weight, mV                                  */
    const uint8_t* syn_d;   /* [S] delay, steps                                */

    /* input lists of the current step (DelayRing.drain's bucket,
     * engine.py:151-163): one append list per group of 32 consecutive neurons,
     * two sets (arrival step & 1): cc_neuron_step(t) delivers step t+1's
     * delay >= 2 events with its idle warps, cc_deliver(t+1) the rest; a record is
     * (spike_ref << 5 | lane) | w_bits << 32.  The delay ring proper is the
     * spike log below: step t delivers the delay-d segment of every spike of
     * step t - d (rows are sorted by delay, network.py:257). */
    int32_t n_groups;       /* ceil(n_local / 32)                              */
    int32_t bin_pad;        /* unused records after each list: list stride is
                               bin_cap + bin_pad (staggers the list starts over
                               L2 slices / DRAM channels)                      */
    uint32_t* bin_cnt;      /* [2][n_groups][n_sub][stride] sub-list fill (word 0) */
    uint64_t* bin_rec;      /* [2][n_groups][n_sub][bin_cap + bin_pad]   */
    uint32_t* grp_n;        /* [n_groups] inputs of the current step per group  */
    uint32_t* grp_sub;      /* [n_groups][n_sub] records kept per sub-list */
    uint32_t* ovf_rec;      /* [2][ovf_cap][4] {group, lane, spike_ref, w_bits} */
    uint32_t* ovf_cnt;      /* [2]                                             */
    uint32_t* ovf_sorted;   /* [ovf_cap][4] overflow of the current step, grouped by group */
    int32_t* ovf_off;       /* [n_groups] start of a group's run in ovf_sorted  */
    int32_t* ovf_fill;      /* [n_groups] grouping cursors (zero between steps) */

    /* spike log (AER payloads, network.py:60-63), one slot per emission step,
     * log_slots = d_max + 1; each entry carries its row start and the row's
     * delay-segment offsets (copied from dseg when the spike is logged) */
    double* log_t;          /* [log_slots][spk_cap]                            */
    uint32_t* log_gid;      /* [log_slots][spk_cap]                            */
    unsigned long long* log_ctr; /* [log_slots] spikes logged                  */
    unsigned long long* log_len; /* [log_slots] sum of their row lengths (the
                               reference's recurrent_events, engine.py:366)     */
    int64_t* log_r0;        /* [log_slots][spk_cap] CSR row start              */
    uint16_t* log_dseg;     /* [log_slots][spk_cap][seg_stride]                */
    const uint16_t* dseg;   /* [n_rows][seg_stride]: dseg[r][d] = synapses of row
                               r with delay <= d (d = 0..d_max), cc_build_dseg */

    /* outputs */
    uint32_t* raster_gid;   /* [raster_cap]                                    */
    double* raster_t;       /* [raster_cap]                                    */
    uint32_t* out_gid;      /* [out_cap] exchange out-list (direct_log == 0)   */
    double* out_t;          /* [out_cap]                                       */
    float* scratch;         /* [scratch_cap][14] spill staging (56 B per event) */
    int32_t* ev_n;          /* [n_local] events staged for each neuron          */
    int32_t* ev_nr;         /* [n_local] of which recurrent                     */
    /* ordered inputs of the step, one 48 B record {t, w, em, ec, f, ecr} each,
     * written by the staging warps and consumed by the group's in-order update */
    double* evrec;          /* [evrec_cap][6]                                    */
    int64_t evrec_cap;
    int32_t* ev_off;        /* [n_local] first record of each neuron this step  */
    uint32_t* grp_items;    /* [n_groups] work items planned for each group     */
    uint32_t* grp_done;     /* [n_groups] items finished (zero between steps)   */
    uint32_t* rounds;       /* [CC_ITEM_CLASSES][round_cap][2] work items {group, l0 | l1 << 8},
                               by size class (class 0 = largest)                */
    int64_t round_cap;
    const int32_t* probe_map; /* [n_local] probe slot or -1                    */
    double* probe_out;      /* [steps][n_probe][5] V c last refr V_end         */
    int64_t probe_steps;    /* rows in probe_out                               */
    cc_ctl* ctl;
    /* [256] counters, each on its own 128 B line (away from the work-item
     * claims in ctl): [0] next step's delay>=2 units claimed by k_stage's idle
     * warps, [32] k_stage warps out of work items, [64] k_stage grid barrier,
     * [96] k_stage work-item claims, [128] its ordered-input record cursor */
    uint32_t* tailc;
    /* [n_local] or NULL: with direct_log, neurons with a destination shard
     * other than this one also go to the exchange out-list (cc_pack_aer) */
    const uint8_t* remote;

    /* peer exchange (NULL xdst: none).  k_stage pushes every spike of a
     * neuron with xmask bit d set into xdst[d]'s region (NVLink stores) and its
     * last block publishes the per-destination counts in the flag words;
     * cc_exchange_ingest waits for every linked source's flag of the step and
     * logs the received spikes (deliver_spikes, network.py:325-379). */
    int32_t n_ranks;        /* entries in xdst / xsrc (<= 32)                   */
    int32_t rank;           /* this shard's rank                                */
    const uint32_t* xmask;  /* [n_local] destination ranks of each neuron (bit d) */
    const cc_xpeer* xdst;   /* [n_ranks] send side (device memory)              */
    const cc_xpeer* xsrc;   /* [n_ranks] receive side (device memory)           */
    uint32_t* xcnt;         /* [32] records pushed per destination this step (zero between steps) */
    int64_t xwait_ns;       /* give up waiting for a source's flag after this long (CC_ERR_XWAIT) */

    /* routed delivery (l1_cnt == NULL: cc_deliver deposits straight into the
     * input lists, one scattered 8 B store per event).  With it, cc_deliver
     * runs two passes, each a counting sort of a tile of events in shared
     * memory followed by coalesced run copies: pass 1 (k_route) routes the
     * step's arrivals to one record array per region of 2^l1_rb consecutive
     * target neurons, pass 2 (k_bin) distributes every region's records to its
     * input lists.  A pass-1 record is 10 B: spike_ref, weight bits, target
     * within the region. */
    int32_t l1_rb;          /* log2 neurons per region (5 .. 16)                 */
    int32_t n_regions;      /* ceil(n_local / 2^l1_rb) <= CC_L1_MAX_REGIONS     */
    int64_t l1_cap;         /* records per region and step                      */
    uint32_t* l1_cnt;       /* [2][n_regions][CC_L1_STRIDE] region fill (word 0), by step parity */
    uint32_t* l1_ref;       /* [n_regions][l1_cap]                              */
    uint32_t* l1_w;         /* [n_regions][l1_cap]                              */
    uint16_t* l1_tgt;       /* [n_regions][l1_cap]                              */
    /* optional (l1_rb <= CC_L1_NCNT_MAX_RB): k_bin also counts the records it
     * stores per target neuron, so that the planning pass takes a neuron's
     * recurrent input count from here instead of reading the group's records;
     * every list record of the step must then come through k_bin (no tail
     * delivery).  The planning pass zeroes what it reads. */
    uint32_t* l1_ncnt;      /* [2][n_groups * 32] records per neuron, by step parity, or NULL */
} cc_shard;

/* ---------------------------------------------------------------- misc */
int cc_abi_version(void);
const char* cc_last_error(void);
/* sizeof(cc_shard) and sizeof(cc_ctl) as compiled, so hosts can verify layout. */
int64_t cc_sizeof_shard(void);
int64_t cc_sizeof_ctl(void);
int64_t cc_sizeof_xpeer(void);

/* CUDA-event timers usable inside captured CUDA graphs (records use
 * cudaEventRecordExternal): per-kernel durations of graph replays. */
int cc_timer_create(int32_t n, void** handle);
int cc_timer_record(void* handle, int32_t i, void* stream);
float cc_timer_elapsed_ms(void* handle, int32_t i, int32_t j);
int cc_timer_destroy(void* handle);

/* ------------------------------------------------------- simulation step */
/* Initial state: V = V_r + u (V_theta - V_r), u = counter_uniforms(seed,
 * INIT_STATE, gid, 0, 0); c = 0, last_t = 0, refr_until = -inf.
 * Replaces engine.py:297-302 and NeuronBlock.__init__ (model.py:263-267). */
int cc_init_state(const cc_shard* sh, void* stream);

/* Step phase (3): deliver the events arriving in step t - the delay-d segment
 * of the row of every spike logged for step t - d, d = 1..d_max - into the
 * step's per-group input lists; adds the row lengths of step t-1's spikes to
 * ctl->rec_events.  Replaces the expand block engine.py:338-367 with
 * DelayRing.insert/drain (engine.py:138-163): the same events reach the same
 * step, expanded at arrival instead of at emission. */
int cc_deliver(const cc_shard* sh, void* stream);

/* One-time launch configuration of the step kernels (shared-memory opt-in,
 * persistent grid size).  Call once before capturing steps into a CUDA graph;
 * cc_neuron_step calls it itself otherwise. */
int cc_prepare(void);

/* Step phases (4)-(6): drain the step's input lists, generate the external
 * Poisson events, order each neuron's inputs by (time, source, weight) and
 * integrate them exactly; emit spikes; idle warps deliver the next step's
 * delay >= 2 events.  Increments ctl->t.
 * Replaces DelayRing.drain (engine.py:151-163), _external_events
 * (engine.py:191-206), the lexsort (engine.py:386) and
 * NeuronBlock.integrate_sorted (model.py:289-337). */
int cc_neuron_step(const cc_shard* sh, void* stream);

/* Multi-shard mode: append the n received AER events (gid, t) emitted in
 * step ctl->t - 1 to the delivery log.  Stands in for the receive half of
 * deliver_spikes (network.py:360-378) + rows_for (network.py:135-141). */
int cc_ingest(const cc_shard* sh, const uint32_t* in_gid, const double* in_t,
              const int32_t* in_n, void* stream);

/* Multi-shard send, device-driven (capturable in a CUDA graph): pack this
 * shard's out-list into one fixed-size slot per destination, selected by the
 * per-neuron destination bit mask (source_masks, network.py:229-230):
 * send[d] = {count, gid_0, t_0 bits, gid_1, ...}, int64, stride 1 + 2 cap.
 * local_of_col maps a global column to its rank among owned columns.  The
 * out-list is consumed (ctl->out_n = 0).  An all-to-all of the slots (equal
 * splits, NCCL) stands in for the counters-then-payloads exchange of
 * deliver_spikes (network.py:325-379). */
int cc_pack_aer(const cc_shard* sh, const uint32_t* dest_mask_by_local, int32_t n_dest,
                int32_t cap, int64_t* send, const int32_t* local_of_col, void* stream);

/* Multi-shard receive of n_src packed slots (same layout): log the received
 * spikes of step ctl->t - 1 that have rows on this shard. */
int cc_ingest_aer(const cc_shard* sh, const int64_t* recv, int32_t n_src, int32_t cap,
                  void* stream);

/* Peer exchange, receive half (capturable; one launch per step after
 * cc_neuron_step): wait until every linked source rank has published its
 * flag for step ctl->t - 1 (acquire, system scope; CC_ERR_XWAIT after
 * sh->xwait_ns), then log its records that have rows on this shard.  With
 * every rank's step kernels finished before the launch (host-synchronised
 * mode, ranks sharing one GPU) the wait returns at once.  Replaces the
 * receive half of deliver_spikes (network.py:360-378) + rows_for
 * (network.py:135-141); the send half is fused into cc_neuron_step. */
int cc_exchange_ingest(const cc_shard* sh, void* stream);

/* Receive windows for the peer exchange: cc_xwin_alloc cudaMallocs `bytes`
 * (zeroed) on the current device and returns the pointer and its 64-byte CUDA
 * IPC handle; cc_xwin_open maps another process's window (peer access enabled
 * lazily); cc_xwin_close / cc_xwin_free release them. */
int cc_xwin_alloc(int64_t bytes, void** ptr, uint8_t* handle64);
int cc_xwin_open(const uint8_t* handle64, void** ptr);
int cc_xwin_close(void* ptr);
int cc_xwin_free(void* ptr);

/* CC_CNT_STRIDE_FOR(n_sub) if the library carries the step kernels for n_sub
 * sub-lists per group (CC_NSUB_A, CC_NSUB_B), else 0. */
int32_t cc_cnt_stride(int32_t n_sub);

/* Kernels cc_deliver + cc_neuron_step launch per step for this shard: 3
 * (k_deliver, k_plan, k_stage), 2 when the planning runs inside k_stage. */
int32_t cc_kernels_per_step(const cc_shard* sh);

/* Warps of k_stage's persistent grid for this shard (SM count x resident blocks
 * per SM x warps per block; depends on d_max and n_sub). */
int32_t cc_stage_warps(const cc_shard* sh);

/* Delay-segment table of a CSR whose rows are sorted by delay: out[r][d] =
 * synapses of row r with delay <= d, d = 0..d_max (u16, row stride `stride`).
 * Sets *err (CC_ERR_DSEG) if a row exceeds 65535 synapses. */
int cc_build_dseg(const int64_t* row_off, const uint8_t* syn_d, int64_t n_rows, int32_t d_max,
                  int32_t stride, uint16_t* out, unsigned* err, void* stream);

/* ------------------------------------------------- connectivity generator */
/* Philox4x64-10 generator of the incoming-synapse CSR of one shard, bit-exact
 * with connectivity.py:383-417 (Bernoulli targets, ziggurat normal weights,
 * uniform / exponential delays), for the sources listed in src_gid.
 * Pass 1 (cc_gen_count) writes the row length of every listed source;
 * the host scans them into row_off; pass 2 (cc_gen_fill) writes the rows,
 * sorted by (delay, layout order) like network.py:257.
 * Layout tables (geometry.layout_blocks): blk_col/blk_p [n_columns][kmax],
 * blk_count [n_columns]; col_local [n_columns] = rank of an owned column or -1. */
typedef struct cc_gen {
    uint64_t seed;
    int32_t n_col, n_exc_col, n_columns, kmax;
    const int32_t* blk_col;
    const double* blk_p;
    const int32_t* blk_count;
    const int32_t* col_local;
    double j_ee, j_ei, j_ie, j_ii, sd_frac;
    int32_t delay_kind;      /* 0 uniform, 1 exponential */
    double d_lo, d_scale;    /* uniform: low, high - low; exponential: scale = mean */
    double dt;
    int32_t d_max;
} cc_gen;

int cc_gen_count(const cc_gen* g, const uint32_t* src_gid, int64_t n_src,
                 int64_t* row_len, unsigned* err, void* stream);
int cc_gen_fill(const cc_gen* g, const uint32_t* src_gid, int64_t n_src,
                const int64_t* row_start, int32_t* syn_tgt, float* syn_w,
                uint8_t* syn_d, unsigned long long* checksum, float* scratch,
                int64_t scratch_per_warp, unsigned* err, void* stream);
/* Warps in the generator's persistent grid (scratch is sized per warp). */
int64_t cc_gen_warps(void);
int64_t cc_sizeof_gen(void);

/* Order-independent checksum of the wire records (network.py:70-88) of the
 * rows of the given sources, in global target ids.  Adds into *checksum. */
int cc_csr_checksum(const int64_t* row_off, const uint32_t* src_gid, int64_t n_src,
                    const int32_t* syn_tgt_global, const float* syn_w,
                    const uint8_t* syn_d, int32_t n_col, int32_t n_exc_col,
                    unsigned long long* checksum, void* stream);

/* Raw stream probes used by the parity tests.  kind: 0 Philox4x64-10 words
 * (bit patterns), 1 random() doubles, 2 ziggurat standard normals,
 * 3 ziggurat exponentials (serial reader); 11 / 12 the warp-cooperative
 * exponential / normal walk of the generator.  Plus
 * counter_uniforms(seed, purpose, a, b, k) of rng.py:74-90. */
int cc_test_philox(uint64_t seed, uint64_t purpose, uint64_t a, int64_t n,
                   int32_t kind, double* out, void* stream);
/* The neuron update's exponentials on n arguments: kind 0 fexp (table-driven
 * e^x), 1 fexpm1, 2 / 3 libdevice exp / expm1 for comparison. */
int cc_test_math(int32_t kind, const double* x, double* out, int64_t n, void* stream);
int cc_test_counter_uniforms(uint64_t seed, uint64_t purpose, const uint64_t* a,
                             uint64_t b, const uint64_t* k, int64_t n, double* out,
                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CORTICARC_B200_H */

/*
 * m2c.h -- C ABI of libm2c: the B200-native (sm_100a) dynamic sparse mixed-precision FFN
 * decode step of M2Cache (arXiv 2410.14740).
 *
 * Citations: P:L = PAPER.md line L (section); DESIGN.md R# = the reading taken where the
 * paper is silent.  The calls follow the paper's statement of the problem
 * (P:73): 1) Active Neuron Identification (m2c_predict_rank), 2) Selective Loading into GPU
 * (m2c_cache_lookup_fill), 3) Active Score-based Quantization (m2c_quant_pack /
 * m2c_load_layer), then the sparse FFN over the mixed-precision active neurons
 * (m2c_sparse_ffn_forward) and the whole-token driver (m2c_decode_step).
 *
 * Conventions (all calls):
 *   - Pointers named *_dev / device buffers are CUDA device pointers; "device or pinned"
 *     pointers may also be page-locked host memory (UVA-mapped).  Pageable host memory is
 *     never accepted except where stated (host-side structs).
 *   - All large memory is CALLER-OWNED (PyTorch allocates it); the library never frees caller
 *     memory.  The context owns only a small workspace (see m2c_create).
 *   - fp16 tensors are IEEE binary16, passed as void* (no CUDA types in the ABI).
 *   - Asynchronous calls are enqueued on the context's compute stream (borrowed from the
 *     caller, who keeps it alive); CUDA errors of enqueued kernels surface as M2C_ERR_CUDA on
 *     the next synchronising call.  Host-side validation happens before any launch; on error
 *     nothing is enqueued.  m2c_last_error() returns a thread-local message.
 *   - F_r = d_ff / shard_count is the rank-local neuron count; neuron ids in every list are
 *     rank-local (global id = shard_index * F_r + local id).
 */
#ifndef M2C_H
#define M2C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define M2C_ABI_VERSION 1

typedef struct m2c_ctx m2c_ctx;
typedef struct CUstream_st *m2c_stream_t; /* == cudaStream_t, borrowed */
typedef struct CUevent_st *m2c_event_t;   /* == cudaEvent_t, borrowed */

typedef enum {
    M2C_OK = 0,
    M2C_ERR_INVALID_ARG = 1, /* null / misaligned pointer, bad bits, bad range */
    M2C_ERR_CONFIG = 2,      /* inconsistent model / plan (e.g. tiers do not sum to k) */
    M2C_ERR_CAPACITY = 3,    /* cache capacity < k_tau, or > the per-pool limit */
    M2C_ERR_CUDA = 4,        /* a CUDA runtime call or kernel failed */
    M2C_ERR_NCCL = 5,        /* NCCL missing or an NCCL call failed */
    M2C_ERR_STATE = 6        /* call order violated (e.g. step not increasing, layer not loaded) */
} m2c_status;

/* Model shape of one rank.  d_model % 256 == 0 and <= 8192 (128-element quantisation groups,
 * R4, and 8-element chunks per thread in the FFN kernel); group == 128; d_ff % shard_count == 0;
 * pred_rank = 16 * 2^j <= 512; act 0 = SiLU, 1 = ReLU (R6).  Violations: M2C_ERR_CONFIG. */
typedef struct {
    int32_t d_model, d_ff, n_layers, pred_rank, group;
    int32_t shard_index, shard_count;
    int32_t act;
} m2c_model_desc;

/* Active set size and its split into FP16 / INT8 / INT4 tiers (R3). */
typedef struct {
    int32_t k, k_fp16, k_int8, k_int4;
} m2c_tier_plan;

/* HBM neuron cache of one layer: mode 0 = resident (all F_r neurons of all tiers in HBM,
 * identity slots), 1 = LRU (R7), 2 = ATU (LRU with cap_slots[t] == k_t).
 * cap_slots[t] = slots of the tier-t pool (t: 0 FP16, 1 INT8, 2 INT4); ignored if resident. */
typedef struct {
    int32_t mode;
    int32_t cap_slots[3];
} m2c_cache_cfg;

/* ---- helpers (pure host functions, no CUDA) -------------------------------------------- */
const char *m2c_last_error(void);
int32_t m2c_abi_version(void);

/* Bytes of one packed neuron record of a tier (R1, R4): FP16 6d; INT8 3d + 9d/128;
 * INT4 3d/2 + 9d/128; each padded to 16 B.  Returns -1 for bad arguments. */
int64_t m2c_record_bytes(int32_t tier_bits, int32_t d_model);

/* R3: k = floor(active_pct * F_r / 100); k16 = floor(k*a16/den); k8 = floor(k*a8/den);
 * k4 = k - k16 - k8.  (25, 25, 100) is the paper's 25/25/50 mix. */
m2c_status m2c_tier_plan_make(int32_t F_r, int32_t active_pct, int32_t a16, int32_t a8,
                              int32_t den, m2c_tier_plan *out);

/* R8: capped LRU sizing.  budget = budget_num/budget_den x FP16 bytes of the layer FFN (6 d F_r);
 * cap_slots[t] = floor(M k_t), M = budget / sum_t k_t nb_t (computed in double). */
m2c_status m2c_cache_cfg_capped(const m2c_model_desc *desc, const m2c_tier_plan *plan,
                                int32_t budget_num, int32_t budget_den, int32_t mode,
                                m2c_cache_cfg *out);

/* Sizes of the caller-owned regions m2c_load_layer needs for one layer: hbm_bytes (device:
 * predictor + tier pools + cache metadata), host_pinned_bytes (pinned host tier: all three
 * tiers packed, LRU/ATU only; 0 if resident).  Each region must be 256-B aligned. */
m2c_status m2c_layer_footprint(const m2c_model_desc *desc, const m2c_cache_cfg *cfg,
                               size_t *hbm_bytes, size_t *host_pinned_bytes);

/* ---- context --------------------------------------------------------------------------- */
/* Device-side invariant violations (non-finite x, a grid-barrier or peer-exchange timeout, an
 * inconsistent selection count) are flagged by the kernels into a pinned host word; the next
 * call on the context that takes it returns M2C_ERR_STATE (without synchronising) and
 * m2c_last_error() names the violation.
 *
 * Creates a context on `device` with borrowed streams `compute` and `copy` (copy carries the
 * miss fills, "dedicated CUDA streams").  `decode_plan` is the plan m2c_decode_step
 * uses.  The context allocates a small device workspace (O(F_r + k + 148 d) bytes). */
m2c_status m2c_create(const m2c_model_desc *desc, int32_t device, m2c_stream_t compute,
                      m2c_stream_t copy, const m2c_tier_plan *decode_plan, m2c_ctx **out);
m2c_status m2c_destroy(m2c_ctx *ctx);

/* ---- a0: pack (P:73 step 3; R1, R4) -------------------------------------- */
/* Packs neurons [n_begin, n_end) of one tier (16, 8 or 4 bits) into `records_out`
 * (n_end - n_begin records of m2c_record_bytes(tier_bits, d) bytes, record i = neuron
 * n_begin + i).  Inputs are neuron-major fp16 [n][d]: W_gate rows, W_up rows, W_down
 * columns (= rows of W_down^T).  Pointers: device or pinned, 16-B aligned.  Bit-exact
 * contract (tests compare every byte with the oracle).  Asynchronous on `stream`. */
m2c_status m2c_quant_pack(int32_t d_model, int32_t tier_bits, const void *w_gate,
                          const void *w_up, const void *w_down_t, int64_t n_begin, int64_t n_end,
                          void *records_out, m2c_stream_t stream);

/* ---- layer load ------------------------------------------------------------------------ */
/* Copies the predictor (pred_A int8 [r][d], pred_B int8 [F_r][r], rank-local rows) into
 * hbm_region, packs the rank's F_r neurons in all three tiers, places them in the HBM pools
 * (resident) or in host_region (LRU/ATU: pinned host tier, "loaded in lower precision
 * from DRAM"; R10), and initialises the cache metadata (identity / cold).  Synchronous: the
 * master weights may be freed when it returns.  Errors: M2C_ERR_CAPACITY if an LRU pool is
 * smaller than the decode plan's k_t or larger than 8192 slots. */
m2c_status m2c_load_layer(m2c_ctx *ctx, int32_t layer, const void *w_gate, const void *w_up,
                          const void *w_down_t, const int8_t *pred_A, const int8_t *pred_B,
                          const m2c_cache_cfg *cfg, void *hbm_region, void *host_region);

/* ---- a1-a3: predictor, top-k, tier split (P:70, P:73 step 1; R2, R3) ---------
 * x: fp16 [d] device.  Outputs (device, any may be NULL except tier_ids):
 *   rank_list int32 [k]   : active ids in rank order (score desc, id asc)
 *   tier_of   int8  [F_r] : -1 inactive, 0 FP16, 1 INT8, 2 INT4
 *   tier_ids  int32 [k]   : three segments [k16 | k8 | k4], ids ascending in each
 *   scores    int32 [F_r] : predictor scores s = B hq
 * Plan must satisfy k16 + k8 + k4 == k <= F_r (else M2C_ERR_CONFIG, host-checked). */
m2c_status m2c_predict_rank(m2c_ctx *ctx, int32_t layer, const void *x,
                            const m2c_tier_plan *plan, int32_t *rank_list, int8_t *tier_of,
                            int32_t *tier_ids, int32_t *scores);

/* ---- a4-a5: cache lookup + asynchronous miss fill (R7, R9) ---
 * Looks the plan's tier segments of tier_ids up in the layer's per-tier pools at timestamp
 * `step` (must strictly increase per layer, else M2C_ERR_STATE).  Outputs (device):
 *   slots      int32 [k]          : pool slot of tier_ids[i]
 *   hit_bitmap uint32 [ceil(k/32)]: bit i set iff tier_ids[i] hit
 *   miss_log   int32 [k][2] or NULL: (id, slot) of misses; tier t's misses start at the
 *                                    segment offset of t (0, k16, k16+k8)
 *   evict_log  int32 [k][2] or NULL: (evicted id, slot), same offsets
 *   counts     int32 [6]  or NULL : misses per tier (3), evictions per tier (3)
 * The lookup runs on the compute stream; the fills run on the copy stream and `fill_done`
 * (caller-created event, may be NULL) is recorded there.  Resident mode: identity slots,
 * every bit set, no fills. */
m2c_status m2c_cache_lookup_fill(m2c_ctx *ctx, int32_t layer, int64_t step,
                                 const int32_t *tier_ids, const m2c_tier_plan *plan,
                                 int32_t *slots, uint32_t *hit_bitmap, int32_t *miss_log,
                                 int32_t *evict_log, int32_t *counts, m2c_event_t fill_done);

/* ---- a6-a7: fused dequant-GEMV + SiLU.mul + sparse down-projection --
 * Computes, for the plan's active neurons, y = sum_n act(g_n) u_n W_down[:, n] reading the
 * records in place in the cache pools ("directly used for inference computation").
 * slots: from m2c_cache_lookup_fill, or NULL in resident mode (slot = id).  hit_bitmap: NULL
 * = everything resident; else hits are computed first, then the compute stream waits on
 * fill_done (if non-NULL) and the misses are computed (R11).  Outputs (device, either may be
 * NULL): y_partial fp32 [d] = this rank's sum before any all-reduce; y fp16 [d] = the
 * all-reduced (if the context has a communicator with >1 rank) sum rounded to fp16.
 * LRU/ATU layers: the hit and miss work lists are the ones the context's most recent
 * m2c_cache_lookup_fill built, so that call must be for THIS layer (no other lookup and no
 * m2c_decode_step in between), else M2C_ERR_STATE. */
m2c_status m2c_sparse_ffn_forward(m2c_ctx *ctx, int32_t layer, const void *x,
                                  const int32_t *tier_ids, const int32_t *slots,
                                  const uint32_t *hit_bitmap, const m2c_tier_plan *plan,
                                  m2c_event_t fill_done, float *y_partial, void *y);

/* ---- multi-GPU (d_ff sharding, R13) ----------------------------------------------------
 * nccl_unique_id: 128 bytes from m2c_nccl_unique_id on rank 0, broadcast by the caller (the
 * torch process group is used for bootstrap only).  nccl_lib: path of libnccl.so.2 (dlopen'd;
 * NULL = default search).  Afterwards every layer all-reduces the fp32 partial sums once
 * (resident stacks: the layer-split k_decode, one launch per layer; LRU/ATU: the kernel
 * chain).  nranks == 1 creates a one-rank communicator: the same engines run with identity
 * collectives (the single-GPU test of the NCCL wiring). */
m2c_status m2c_nccl_unique_id(const char *nccl_lib, void *id_out_128);
m2c_status m2c_comm_init(m2c_ctx *ctx, int32_t nranks, int32_t rank, const void *nccl_unique_id,
                         const char *nccl_lib);

/* ---- §8(e): the all-reduce fused into the whole-token kernel over peer memory -----------
 * For a d_ff-sharded resident stack ("fused all-reduce inside the FFN kernel via
 * NVLink P2P stores"), k_decode can exchange each layer's reduced y chunks itself instead of
 * the layer-split engine's NCCL all-reduce: in its reduction phase the CTA owning a 32-wide
 * chunk of d stores the chunk into every rank's exchange buffer (peer stores over NVLink) as
 * 8-byte (round flag << 32 | f32) words, polls until the P words of each element in its own
 * buffer carry this round's flag, and sums them in rank order 0..P-1 (so results equal a host
 * emulation of the rank-order sum, not necessarily NCCL's order).  No fences, no counters, no
 * cross-GPU barrier: only the P CTAs owning the same chunk meet.
 *   m2c_p2p_buffer: allocates this rank's exchange buffer (device, zeroed; owned by the
 *     context): [2][P][d] u64 | u32 rounds.  dev_ptr_out: its address; ipc_handle_out (64 B,
 *     nullable): a cudaIpcMemHandle for other processes.
 *   m2c_p2p_connect: dev_ptrs [P] (same process: device pointers the contexts' GPUs can
 *     access) or ipc_handles [P][64] (other processes; opened here, closed by m2c_destroy).
 *     nranks must equal shard_count (>= 2).  All ranks must run m2c_decode_step on the same
 *     tokens with the same grid (m2c_set_grid) and be co-resident on their GPUs; a rank that
 *     waits > 5 s for a peer sets error bit 16 and continues (wrong result, never a hang).
 *   m2c_set_grid: CTAs of the context's kernels, 1..SM count (default: SM count).  Two ranks
 *     sharing one GPU (the single-GPU test of this path) use half the SMs each.  Synchronises
 *     the compute stream and resets the decode kernel's grid-barrier counter. */
m2c_status m2c_p2p_buffer(m2c_ctx *ctx, uint64_t *dev_ptr_out, void *ipc_handle_out);
m2c_status m2c_p2p_connect(m2c_ctx *ctx, int32_t nranks, const uint64_t *dev_ptrs,
                           const void *ipc_handles);
m2c_status m2c_set_grid(m2c_ctx *ctx, int32_t ctas);

/* ---- whole token (all layers), CUDA-graph captured ------------------------------------
 * x_inout: fp16 [d] device; on return (asynchronously) holds x_L where
 * x_{l+1} = fp16(x_l + fp16(y_l)) (R14).  step: strictly increasing (LRU timestamps). */
m2c_status m2c_decode_step(m2c_ctx *ctx, void *x_inout, int64_t step);

/* The tier lists the last m2c_decode_step selected for layer `layer` (any cache mode): int32
 * [k], three ascending segments k16 | k8 | k4 (the layout of m2c_predict_rank's tier_ids),
 * written to the device buffer tier_ids_out on the compute stream.  M2C_ERR_STATE before the
 * first decode step; M2C_ERR_CAPACITY if a tier has more than 32768 entries. */
m2c_status m2c_decode_lists(m2c_ctx *ctx, int32_t layer, int32_t *tier_ids_out);

/* Parity trace (the replay harness): with device buffers x_trace fp16
 * [n_layers + 1][d] and y_trace fp32 [n_layers][d] set (caller-owned; NULL, NULL disables),
 * every later m2c_decode_step also writes each layer's input x_l, the final x_L, and each
 * layer's output y_l (after the all-reduce when sharded) before its fp16 rounding.  Every
 * engine writes the same quantities; the decode graph is re-captured. */
m2c_status m2c_set_trace(m2c_ctx *ctx, void *x_trace, float *y_trace);

/* LRU/ATU pool state of (layer, tier) (R7, oracle O7): occupant_out int32 [cap] (-1 = empty)
 * and last_out int32 [cap] (step of the last use, -1 = never), device buffers (either may be
 * NULL), copied asynchronously on the compute stream; *cap_out = the pool's slot count.
 * M2C_ERR_STATE for a resident layer. */
m2c_status m2c_cache_state(m2c_ctx *ctx, int32_t layer, int32_t tier, int32_t *occupant_out,
                           int32_t *last_out, int32_t *cap_out);

/* Disables (0) or enables (1, default) CUDA-graph capture of m2c_decode_step. */
m2c_status m2c_set_graph(m2c_ctx *ctx, int32_t enable);

/* m2c_decode_step engine.  1 (default): a stack whose layers are all resident, unsharded
 * (no communicator), with F_r <= 40960 and ceil(F_r / SMs) <= d_model / 8 runs as ONE
 * persistent cooperative kernel per token
 * (k_decode: one CTA per SM, grid barriers between the phases of a layer, L2 lookahead of the
 * next layer's predictor slices and of the records the previous token selected for it --
 * adjacent tokens share ~80% of their active neurons); other stacks run the per-phase
 * kernel chain with the same L2 prefetch hint.  0: the per-phase kernel chain, no prefetch.
 * Results are bit-identical either way (tests). */
m2c_status m2c_set_fused(m2c_ctx *ctx, int32_t enable);

/* Phase timing.  m2c_profile(ctx, 1) instruments m2c_decode_step (the graph is re-captured):
 * the kernel chain records 5 CUDA events per layer (before predict | after predict | after
 * select | after cache+FFN | after reduce); k_decode records globaltimer stamps per (layer,
 * CTA).  m2c_profile_read synchronises the compute stream and writes, for the last decode
 * step, ms[l*4 + {0,1,2,3}] = predictor, select, cache lookup + FFN, reduce/all-reduce/residual
 * of layer l (k_decode: measured on the slowest CTA, barriers included in the phase they
 * end).  ffn_launches_out = FFN kernel launches per layer (0 for k_decode).
 * m2c_profile_stamps copies k_decode's raw stamps, uint64 ns [n_layers][G][M2C_DECODE_STAMPS]
 * (0 layer start, 20/21/22 P2 sub-steps (h max, hq, scores), 1 scores + sorted run done,
 * 4 after barrier Bs, 2/3/16/10 select sub-steps (runs in smem,
 * cut bins, candidates, exact cuts), 18/19/11 list sub-steps, 5 select done, 14/15 FFN
 * sub-steps, 6 FFN done, 7 after barrier By, 8 reduction + next h done, 9 kernel end,
 * 12/13 prologue start / end (layer 0); stamps not listed are unused and hold garbage);
 * *n_out = the element count (out may be null to query it); M2C_ERR_STATE if the last step
 * did not run on k_decode with profiling. */
#define M2C_DECODE_STAMPS 24
m2c_status m2c_profile(m2c_ctx *ctx, int32_t enable);
m2c_status m2c_profile_read(m2c_ctx *ctx, float *ms, int32_t *ffn_launches_out);
/* Miss-fill duration of each LRU/ATU layer in the last profiled m2c_decode_step (ms, copy
 * stream, CUDA events around the fill kernels; 0 for resident layers).  M2C_ERR_STATE if
 * profiling is off or the last step ran k_decode alone (no fills). */
m2c_status m2c_profile_fill(m2c_ctx *ctx, float *ms_per_layer);
m2c_status m2c_profile_stamps(m2c_ctx *ctx, uint64_t *out, int64_t cap, int64_t *n_out);
/* m2c_profile_events: the last decode step's per-layer CUDA-event timeline (kernel-chain
 * engines: resident chain, LRU/ATU), ms since layer 0's first mark, [n_layers][11]: compute
 * stream 0 layer start, 1 predictor done, 2 select done, 3 FFN done, 4 reduce done; copy stream
 * 5 miss fill start, 6 miss fill end; compute stream (early-fill LRU engine) 7 LRU update done,
 * 8 hit FFN done, 9 miss queue done, 10 requantisation done (-1: not recorded).  The copy-versus-compute overlap of the LRU engine (P:11,
 * P:396) is read from it.  *n_out = n_layers * 11 (out may be null);
 * M2C_ERR_STATE if profiling is off or the last step was one k_decode launch. */
m2c_status m2c_profile_events(m2c_ctx *ctx, float *out, int64_t cap, int64_t *n_out);

/* Kernels launched by the last m2c_decode_step (per token), and cumulative cache counters
 * (hits, misses per tier) since the last reset (device counters; synchronises). */
/* ---- NEXT-3: exact global top-k under d_ff sharding --------------
 * Shard-local top-k (R13) keeps k_r per rank; the paper's semantics is one global top-k over
 * all F neurons.  m2c_predict_candidates(ctx, layer, x, n_cand, keys_out): this rank's scores
 * and its top n_cand neurons as int64 keys (score << 32 | ~global id) sorted descending, i.e.
 * (score desc, global id asc) order (R3); device [n_cand].  After an all-gather of every rank's
 * keys into keys_all [P][n_cand] (rank order), m2c_select_global(ctx, keys_all, n_cand,
 * global_plan, tier_ids_out, counts_out) finds the three global cuts (k16, k16+k8, k of the
 * global plan) and writes THIS rank's selected neurons: tier_ids_out [global k] in three
 * segments at the global plan's offsets (0, k16, k16+k8), local ids ascending in each, and
 * counts_out [3] (device) = how many of each tier this rank owns.  Exact (the union over ranks
 * equals the unsharded selection) when n_cand >= min(F_r, k); else M2C_ERR_CONFIG.  P x n_cand
 * x 8 B must fit 200 KiB (M2C_ERR_CAPACITY).  Both calls are asynchronous on the compute
 * stream; the all-gather is the caller's (ncclAllGather over the torch process group). */
m2c_status m2c_predict_candidates(m2c_ctx *ctx, int32_t layer, const void *x, int32_t n_cand,
                                  int64_t *keys_out);
m2c_status m2c_select_global(m2c_ctx *ctx, const int64_t *keys_all, int32_t n_cand,
                             const m2c_tier_plan *global_plan, int32_t *tier_ids_out, int32_t *counts_out);
/* m2c_set_global_topk(ctx, global_plan): the resident, d_ff-sharded m2c_decode_step uses the
 * global selection per layer (the two calls above with ncclAllGather of P x min(F_r, k) int64
 * keys on the compute stream, then the FFN over this rank's part, the all-reduce as before);
 * NULL restores shard-local top-k (R13).  Needs m2c_comm_init with an NCCL that exports
 * ncclAllGather.  (Validated on one GPU through the two calls with emulated all-gathers; the
 * NCCL wiring itself needs >= 2 GPUs.) */
m2c_status m2c_set_global_topk(m2c_ctx *ctx, const m2c_tier_plan *global_plan);

/* ---- NEXT-2: cross-layer lookahead ("the next one layer ... almost 100%") ---------
 * m2c_set_lookahead(ctx, 1): in the LRU/ATU decode chain, after layer l's cache lookup the
 * library also runs layer l+1's predictor and select on x_l (a prediction of layer l+1's
 * selection), marks the predicted neurons that would miss in layer l+1's pools now, and copies
 * their records from the host tier into device staging buffers on the copy stream, overlapped
 * with the rest of layer l.  At layer l+1 a miss whose record was staged is filled device to
 * device.  The selection, the cache state and every output are unchanged (the staging only
 * moves the PCIe transfer earlier); mispredicted records cost extra PCIe traffic.  Not used
 * with an SSD store attached.  Allocates the staging buffers (2 x sum_t k_t nb_t + O(F_r)).
 * m2c_lookahead_stats: misses filled from staging so far (reset: zero it). */
m2c_status m2c_set_lookahead(m2c_ctx *ctx, int32_t enable);
m2c_status m2c_lookahead_stats(m2c_ctx *ctx, int64_t *staged_fills, int32_t reset);

/* ---- a5 fill source: GPU requantisation of tier-churn misses (early-fill LRU/ATU engine) --
 * A neuron selected in the INT8 or INT4 tier that misses that tier's pool but whose FP16
 * record is resident in the layer's FP16 pool (it was active in the FP16 tier recently: ranks
 * move across the tier cuts from token to token) gets its record by quantising
 * the resident FP16 record on the GPU with the offline pack's function (R4, bit-identical to
 * the host tier's record, O0) instead of a PCIe copy ("reduce the data movement").  The
 * miss is still a miss: the cache state, the hit / miss / eviction counts and the outputs are
 * unchanged; only the bytes crossing PCIe shrink.  On by default (decode engine only; the
 * per-call m2c_cache_lookup_fill always copies from the host tier).
 *   m2c_set_requant(ctx, 0 / 1): off / on (invalidates the captured decode graph).
 *   m2c_requant_stats(ctx, out[3], reset): requantised fills per tier so far (out[0] = 0). */
m2c_status m2c_set_requant(m2c_ctx *ctx, int32_t enable);
m2c_status m2c_requant_stats(m2c_ctx *ctx, int64_t *requant_fills, int32_t reset);

/* ---- NEXT-1: SSD -> DRAM tier (§5.4) -----------------
 * The paper keeps the whole model on SSD and stages it into DRAM layer-wise with a two-level
 * DRAM cache: a FIXED area holding the first n layers and a DYNAMIC area managed FIFO, filled
 * by I/O threads at least two layers ahead.  Here:
 *   m2c_store_write(ctx, path): after every layer was loaded in LRU/ATU mode, writes the host
 *     tier (each layer's three packed tiers, verbatim) to a layer-major file, each layer padded
 *     to m2c_store_frame_bytes.  Synchronous.
 *   m2c_store_attach(ctx, path, n_fixed, n_dynamic, lookahead, frames, frames_bytes): from now
 *     on the miss fills read the file-backed DRAM frames instead of the in-memory host tier
 *     (the caller may free that after attaching).  frames: caller-owned pinned host memory of
 *     >= (n_fixed + n_dynamic) x m2c_store_frame_bytes bytes, 4 KiB aligned for O_DIRECT reads.
 *     Layers [0, n_fixed) are read once into the fixed area; one I/O thread keeps layers up to
 *     `lookahead` ahead of the decode loop in the dynamic frames (FIFO), and synchronises on
 *     the GPU's last read of a frame before reusing it.  m2c_decode_step then runs eagerly
 *     (no CUDA graph) and the host blocks in it while a needed layer is still being read.
 *     Outputs are identical to the in-memory host tier (same bytes).
 *   m2c_store_stats: bytes read, layer loads, seconds in reads (I/O thread) and seconds the
 *     decode loop waited for a layer.  m2c_store_detach: stops the I/O thread.
 * Errors: M2C_ERR_STATE (layers not loaded in LRU/ATU mode, short file, read failure),
 * M2C_ERR_CAPACITY (frames too small), M2C_ERR_CONFIG (bad counts). */
size_t m2c_store_frame_bytes(const m2c_model_desc *desc, const m2c_cache_cfg *cfg);
m2c_status m2c_store_write(m2c_ctx *ctx, const char *path);
m2c_status m2c_store_attach(m2c_ctx *ctx, const char *path, int32_t n_fixed, int32_t n_dynamic,
                            int32_t lookahead, void *frames, size_t frames_bytes);
m2c_status m2c_store_detach(m2c_ctx *ctx);
m2c_status m2c_store_stats(m2c_ctx *ctx, int64_t *bytes_read, int64_t *layer_loads, double *io_seconds,
                           double *stall_seconds);

m2c_status m2c_stats(m2c_ctx *ctx, int64_t *kernels_per_token, int64_t hits[3], int64_t misses[3],
                     int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* M2C_H */

// m2c_internal.cuh -- shared internals of libm2c (context, PTX wrappers, launch helpers).
// Part of the PRODUCT path.  Shares nothing with oracle/ (see DESIGN.md §3).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/m2c.h"

namespace m2c {

// ----------------------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------------------
void set_error(const std::string &msg);
m2c_status fail(m2c_status st, const std::string &msg);
m2c_status cuda_fail(cudaError_t e, const char *what);

#define M2C_CUDA(call)                                                   \
    do {                                                                 \
        cudaError_t _e = (call);                                         \
        if (_e != cudaSuccess) return ::m2c::cuda_fail(_e, #call);      \
    } while (0)

constexpr int kMaxPoolSlots = 8192;  // LRU / ATU pool limit (single-CTA bitonic victim sort)
constexpr int kSelectThreads = 1024;
constexpr int kDecodeStamps = M2C_DECODE_STAMPS;  // k_decode profiling stamps per (layer, CTA)
// h = A x accumulators are int64 words kHStride apart (one 256-B L2 line each): every CTA
// adds its column-slice partial sums with red.add.u64, and a packed [r] array would put all
// r counters into a handful of L2 slices whose atomic units serialise them
constexpr int kHStride = 32;

// ----------------------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------------------
struct LayerState {
    bool loaded = false;
    int mode = 0;  // 0 resident, 1 lru, 2 atu
    int cap[3] = {0, 0, 0};
    const int8_t *A = nullptr;  // A^T: [d][r] (column j of the low-rank factor A is row j)
    const int8_t *B = nullptr;  // [F_r][r]
    uint8_t *pool[3] = {nullptr, nullptr, nullptr};
    int32_t *occupant[3] = {nullptr, nullptr, nullptr};
    int32_t *last[3] = {nullptr, nullptr, nullptr};
    int32_t *slot_of[3] = {nullptr, nullptr, nullptr};
    int32_t *ord[3] = {nullptr, nullptr, nullptr};  // LRU order: slots by (last_use, slot)
    const uint8_t *host_rec[3] = {nullptr, nullptr, nullptr};
    const uint8_t *host_base = nullptr;  // the layer's host-tier region (the store's unit)
    size_t host_off[3] = {0, 0, 0};      // tier offsets inside it
    size_t host_bytes = 0;
    int64_t last_step = INT64_MIN;
};

struct NcclApi;  // dlopen'd NCCL entry points


struct Workspace {
    long long *h = nullptr;        // [r][kHStride]: h_i = (A x)_i at h[i * kHStride] (R2)
    int32_t *s = nullptr;          // [F_r]
    int32_t *tier_ids = nullptr;   // [F_r]
    int8_t *tier_of = nullptr;     // [F_r]
    int32_t *slots = nullptr;      // [F_r]
    uint32_t *hit_bits = nullptr;  // [F_r/32 + 1]
    int32_t *hit_items = nullptr;  // [F_r]  compacted hit slots, tier segments
    int32_t *miss_items = nullptr; // [F_r]  compacted miss slots, tier segments
    int32_t *miss_ids = nullptr;   // [F_r]  compacted miss ids (fill source), tier segments
    int32_t *counts = nullptr;     // [16]: 0..2 plan counts, 4..6 hits, 8..10 misses, 12..14 evictions
    float *partial = nullptr;      // [2][G][d]
    float *y32 = nullptr;          // [d]
    __half *xbuf = nullptr;        // [d]
    unsigned long long *stats = nullptr;  // [16] hits[3], misses[3], staged fills, -, requantised
                                          // fills per tier [8..10] (cumulative)
    uint32_t *err = nullptr;       // device error flag word; err + 2 holds the host mirror's
                                   // device address (flag_error)
};

}  // namespace m2c

struct m2c_ctx {
    m2c_model_desc desc{};
    int F_r = 0;
    int device = 0;
    int num_sms = 148;
    cudaStream_t compute = nullptr, copy = nullptr;
    m2c_tier_plan plan{};
    int64_t nb[3] = {0, 0, 0};
    std::vector<m2c::LayerState> layers;
    void *ws_mem = nullptr;
    size_t ws_bytes = 0;
    m2c::Workspace ws;
    int G = 148;              // FFN grid (persistent CTAs)
    cudaEvent_t ev_lookup = nullptr, ev_fill = nullptr, ev_stage = nullptr;
    // decode graph
    bool use_graph = true;
    cudaGraphExec_t graph = nullptr;
    void *graph_x = nullptr;
    int64_t kernels_per_token = 0;
    int64_t launch_counter = 0;
    // phase timing events (m2c_profile): 5 per layer
    std::vector<cudaEvent_t> prof_ev;
    // fused decode-path select: score histogram (s + sel_smax) >> sel_sh into 4096 bins,
    // and the previous token's tier lists per layer (L2 prefetch hint)
    int sel_smax = 0, sel_sh = 0;
    int *ghist = nullptr;       // [2][4096] (the chain uses [0]; k_decode alternates by layer)
    int32_t *prev_ids = nullptr;  // [n_layers][k]
    unsigned long long *sel_status = nullptr;  // [select blocks] decoupled look-back words
    int *sel_done = nullptr;    // select completion counter
    int *sel_epoch = nullptr;   // select launch epoch
    bool use_fused = true;
    bool force_split = false;   // layer-split k_decode even unsharded (testing; m2c_set_fused(ctx, 2))
    bool last_token_split = false;
    // persistent decode kernel (k_decode): layer pointer table, grid-barrier flags, stamps
    void *dec_layers = nullptr;
    unsigned *bar_flags = nullptr;   // [G]
    unsigned *bar_epoch = nullptr;
    unsigned long long *dec_prof = nullptr;  // [n_layers][G][kDecodeStamps]
    int *dec_bin_sh = nullptr;       // [n_layers] k_decode histogram scale per layer
    long long *dec_hb = nullptr;     // [2][r][kHStride] k_decode h accumulators (layer parity)
    unsigned long long *dec_bucket = nullptr;  // [2][4096][128] k_decode rank keys per score bin
    int *dec_sdump = nullptr;        // [F_r] k_decode scores of the current layer
    int *dec_hist = nullptr;         // [2][4096] k_decode score histograms
    unsigned *dec_sabs = nullptr;    // [G] per-CTA max |s| scratch
    bool dec_table_dirty = true;
    bool last_token_fused = false;
    bool decoded = false;            // at least one m2c_decode_step enqueued
    // NEXT-1: SSD -> DRAM store (store.cu); null = the in-memory pinned host tier
    void *store = nullptr;
    // NEXT-2: cross-layer lookahead staging (LRU/ATU decode chain); buffers by layer parity
    bool lookahead = false;
    void *stage_mem = nullptr;
    int32_t *stage_of[2] = {nullptr, nullptr};   // [3][F_r]
    uint8_t *stage_buf[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    int32_t *stage_sid[2] = {nullptr, nullptr};  // [k]
    int32_t *spec_ids = nullptr;                 // [k] predicted tier lists of the next layer
    cudaStream_t stage_stream = nullptr;          // staging copies (own stream: concurrent with fills)
    cudaEvent_t ev_staged[2] = {nullptr, nullptr};  // layer parity: staging complete
    // NEXT-3: exact global top-k in the sharded decode chain
    bool global_topk = false;
    m2c_tier_plan gplan{};
    long long *gkeys = nullptr;   // [n] own candidates | [P][n] gathered
    int32_t *gids = nullptr;      // [k_global] this rank's part of the global tier lists
    // early fill (decode engine, LRU/ATU layers): miss queue, identity list, staging area
    int32_t *mq = nullptr;        // [16 + k]: q[8 + t] = misses of tier t; ids from q + 16
    int32_t *ident = nullptr;     // [k]: ident[seg_t + m] = m
    int32_t *mq_src = nullptr;    // [k]: FP16-pool slot of an INT miss filled by requantisation, or -1
    int32_t *mq_job = nullptr;    // [k]: the requantisation jobs' queue entries (per tier segment)
    int32_t *mq_ready = nullptr;  // [k]: staging entry landed (fill_tag(step, layer)), per tier segment
    cudaStream_t rq_stream = nullptr;  // the requantisation (off the compute chain)
    cudaEvent_t ev_rq = nullptr;
    bool requant = true;          // early-fill engine: INT misses from resident FP16 records
    uint8_t *mstage[3] = {nullptr, nullptr, nullptr};  // [k_t][nb_t]
    void *early_mem = nullptr;
    bool early_fill = true;
    cudaEvent_t ev_q = nullptr, ev_scat = nullptr;
    // §8(e): in-kernel all-reduce over peer memory (m2c_p2p_*)
    bool p2p = false;
    void *p2p_mem = nullptr;          // this rank's exchange buffer [2][P][d] (flag|f32) u64 | rounds
    size_t p2p_bytes = 0;
    unsigned long long *const *p2p_xtab = nullptr;  // device [P] table
    unsigned *p2p_rounds = nullptr;
    void *p2p_tabs = nullptr;
    std::vector<void *> p2p_opened;   // IPC-opened peer bases (closed at destroy)
    // parity trace (m2c_set_trace): x_l [L+1][d] fp16, y_l [L][d] f32, caller-owned
    __half *trace_x = nullptr;
    float *trace_y = nullptr;
    // device error flag mirrored into pinned host memory (checked by every host call)
    uint32_t *err_host = nullptr;
    // early-fill engine: the last layer's scatter (copy stream) still reads the miss lists
    bool scat_pending = false;
    // LRU engine: the last k_reduce also formed the next layer's h (enqueue-time state)
    bool h_prepared = false;
    // per-call API: layer whose hit / miss lists the last m2c_cache_lookup_fill left in ws
    int ws_lists_layer = -1;
    bool fill_pending = false;        // per-call API: a miss fill still reads the ws miss lists
    cudaEvent_t ev_fill_api = nullptr;
    // multi-GPU
    m2c::NcclApi *nccl = nullptr;
    void *comm = nullptr;
    int nranks = 1, rank = 0;
};

namespace m2c {

// ----------------------------------------------------------------------------------------
// launchers (defined in the kernel .cu files); all enqueue on `st`, PDL-enabled
// ----------------------------------------------------------------------------------------
cudaError_t launch_pack(int d, int bits, const __half *g, const __half *u, const __half *dn,
                        int64_t n0, int64_t n1, uint8_t *out, cudaStream_t st);
// L2 prefetch hint: the previous token's tier lists of this layer (resident pools, ids = slots)
struct PrefetchArgs {
    const int32_t *prev_ids = nullptr;  // [k] or null
    const uint8_t *pool[3] = {nullptr, nullptr, nullptr};
    int nb[3] = {0, 0, 0};
    int k[3] = {0, 0, 0};
    int F_r = 0;
};
cudaError_t launch_transpose_i8(int r, int d, const int8_t *A, int8_t *At, cudaStream_t st);
cudaError_t launch_predict(m2c_ctx *c, const LayerState &L, const __half *x, int32_t *scores,
                           int *hist, const int32_t *prefetch_ids, cudaStream_t st);
cudaError_t launch_select(m2c_ctx *c, const int32_t *scores, int *hist, const m2c_tier_plan &p,
                          int32_t *rank_list, int8_t *tier_of, int32_t *tier_ids, cudaStream_t st);
size_t select_smem_bytes(int sh);
// NEXT-3 (k_select.cu)
cudaError_t launch_cand_keys(m2c_ctx *c, const int32_t *scores, const int32_t *rank_list, int n,
                             long long *keys, cudaStream_t st);
cudaError_t launch_select_global(m2c_ctx *c, const long long *keys, int n, const m2c_tier_plan &g,
                                 int32_t *tier_ids, int32_t *counts, cudaStream_t st);
int select_blocks(int F_r);
cudaError_t launch_missq(m2c_ctx *c, const LayerState &L, int32_t *tier_ids, const m2c_tier_plan &p,
                         cudaStream_t st, int32_t *qsrc = nullptr, bool sort = false, bool requant = false);
cudaError_t launch_requant(m2c_ctx *c, const LayerState &L, const m2c_tier_plan &p, cudaStream_t st);
cudaError_t launch_copy_recs(m2c_ctx *c, const uint8_t *const src[3], uint8_t *const dst[3],
                             const m2c_tier_plan &p, const int32_t *counts, const int32_t *srci,
                             const int32_t *dsti, cudaStream_t st, const int32_t *skip = nullptr,
                             int ready_layer = -1);  // ready_layer >= 0: publish mq_ready per record
cudaError_t launch_lru(m2c_ctx *c, LayerState &L, const int32_t *step_dev, const int32_t *tier_ids,
                       const m2c_tier_plan &p, int32_t *slots, uint32_t *hit_bits,
                       int32_t *miss_log, int32_t *evict_log, cudaStream_t st);
cudaError_t launch_fill(m2c_ctx *c, const LayerState &L, const m2c_tier_plan &p, cudaStream_t st,
                        int stage_par = -1);
// NEXT-2 lookahead staging (k_cache.cu): Ln = layer l+1, par = (l+1) & 1
cudaError_t launch_stage_plan(m2c_ctx *c, const LayerState &Ln, int par, const int32_t *spec_ids, cudaStream_t st);
cudaError_t launch_stage_fill(m2c_ctx *c, const LayerState &Ln, int par, cudaStream_t st);
cudaError_t launch_stage_clear(m2c_ctx *c, const LayerState &Ln, int par, cudaStream_t st);
// store.cu (NEXT-1)
m2c_status store_open(m2c_ctx *c, const char *path, int n_fixed, int n_dyn, int ahead, void *frames,
                      size_t frames_bytes, size_t layer_bytes);
void store_close(m2c_ctx *c);
uint8_t *store_acquire(m2c_ctx *c, int l);
void store_release(m2c_ctx *c, int l, cudaStream_t st);
void store_stats(m2c_ctx *c, int64_t *bytes, int64_t *loads, double *io_s, double *stall_s);
m2c_status store_write(m2c_ctx *c, const char *path, size_t layer_bytes);
cudaError_t launch_ffn(m2c_ctx *c, const LayerState &L, const __half *x, const int32_t *items,
                       const int32_t *counts, const m2c_tier_plan &p, float *partial,
                       cudaStream_t st, int wait_layer = -1);  // wait_layer: the early-fill miss FFN
cudaError_t launch_reduce(m2c_ctx *c, int n_partials, const float *partial, const __half *x,
                          float *y32, __half *y16, __half *x_next, int *hist_zero, cudaStream_t st,
                          const int8_t *At_next = nullptr);  // At_next: + the next layer's h (LRU engine)
cudaError_t launch_finalize(m2c_ctx *c, const float *y32, const __half *x, __half *y16,
                            __half *x_next, cudaStream_t st);
// persistent decode kernel (k_decode.cu)
cudaError_t launch_decode(m2c_ctx *c, __half *x, unsigned long long *prof, cudaStream_t st, int layer0 = 0,
                          int nl = -1, const float *pre_y = nullptr, float *post_y = nullptr,
                          int32_t *lists_out = nullptr,  // lists_out: select-only (one layer)
                          bool h_ready = false);  // select-only: h and the histogram prepared by k_reduce
cudaError_t init_decode_attrs();
cudaError_t decode_write_layer_table(m2c_ctx *c, void *dev_table);
size_t decode_layer_table_bytes(int n_layers);
size_t decode_hist_bytes();
size_t decode_bucket_bytes();
bool decode_shape_ok(const m2c_ctx *c);
int sort_tiers_max();
// rank-order tier lists -> ascending ids per tier segment, in place (k_decode.cu)
cudaError_t launch_sort_tiers(m2c_ctx *c, int32_t *ids, const m2c_tier_plan &p, cudaStream_t st);
cudaError_t init_select_attrs();
cudaError_t init_cache_attrs();
cudaError_t init_ffn_attrs();
cudaError_t launch_fill_i32(int32_t *p, int32_t v, int64_t n, cudaStream_t st);
cudaError_t launch_set_counts(int32_t *dst, int32_t a, int32_t b, int32_t c, cudaStream_t st);
cudaError_t launch_iota(int32_t *p, int64_t n, cudaStream_t st);

// PDL-enabled launch (programmatic stream serialization): the dependent kernel calls
// griddep_wait() before touching its predecessor's outputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool pdl = !(getenv("M2C_PDL") && getenv("M2C_PDL")[0] == '0');  // (A/B knob)
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ----------------------------------------------------------------------------------------
// device helpers
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ void griddep_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void griddep_launch() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// one non-blocking probe of an mbarrier phase
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// 1-D bulk copy global -> shared (TMA engine; SASS UBLKCP), completion on an mbarrier.
// EVICT_FIRST L2 policy: the neuron records are streamed once per token.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// bulk L2 prefetch (no smem destination); size multiple of 16, address 16-B aligned
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes & ~15u) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// O3 (R2): exact round-half-up of 127 a / M for 0 <= a <= M < 2^62, i.e.
// floor((254 a + M) / (2 M)).  The fp64 estimate is within one of the answer; two 128-bit
// integer checks pin it.
__device__ __forceinline__ int quant127_u64(unsigned long long a, unsigned long long M) {
    if (M == 0) return 0;
    int q = (int)fma((double)a, 127.0 / (double)M, 0.5);
    q = q < 0 ? 0 : (q > 127 ? 127 : q);
    // q is right iff (2q - 1) M <= 254 a < (2q + 1) M; products as (hi, lo) 128-bit pairs
    const unsigned long long al = a * 254ull, ah = __umul64hi(a, 254ull);
    auto lt = [&](unsigned long long k) {  // 254 a < k M ?
        const unsigned long long ml = M * k, mh = __umul64hi(M, k);
        return ah < mh || (ah == mh && al < ml);
    };
    if (!lt((unsigned long long)(2 * q + 1))) q += 1;
    else if (q > 0 && lt((unsigned long long)(2 * q - 1))) q -= 1;
    return q;
}
// x_j 2^24 as an exact integer (O1): mantissa m (signed, |m| < 2^11) and shift sh, X = m << sh.
// Inf / NaN: m = 0 and *bad set.
__device__ __forceinline__ void fp16_fixed(unsigned b, int &m, int &sh, bool &bad) {
    const int e = (b >> 10) & 31;
    m = b & 1023;
    sh = 0;
    if (e == 31) {
        bad = true;
        m = 0;
    } else if (e) {
        m |= 1024;
        sh = e - 1;
    }
    if (b & 0x8000) m = -m;
}
// Device-side invariant violation: set `bit` in the context's device error word and mirror
// it into the pinned host word whose address the context stores right after it (ws.err + 2),
// so the NEXT host call on the context returns M2C_ERR_STATE without synchronising
// (SURVEY §8(b)).  err bits: 1 non-finite x, 4 grid-barrier timeout, 8 select count
// mismatch, 16 p2p exchange timeout.
// Bounds-checked build (-DM2C_CHECKS=1, tests/test_gpu_checked.py): index and capacity
// invariants at the kernels' computed addresses trap (the launch fails) instead of corrupting
// memory -- the stand-in for compute-sanitizer, which this GPU pool refuses.  Compiled out of
// the product build.
#ifndef M2C_CHECKS
#define M2C_CHECKS 0
#endif
#if M2C_CHECKS
#define M2C_CHECK(c)                                                                         \
    do {                                                                                     \
        if (!(c)) {                                                                          \
            printf("m2c check failed: %s (%s:%d, block %d thread %d)\n", #c, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                       \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define M2C_CHECK(c) \
    do {             \
    } while (0)
#endif
__device__ __forceinline__ void flag_error(uint32_t *err, unsigned bit) {
    atomicOr(err, bit);
    uint32_t *mirror = *reinterpret_cast<uint32_t *const *>(err + 2);
    if (mirror) *reinterpret_cast<volatile uint32_t *>(mirror) = 0x80000000u | bit;
}
// the per-(step, layer) value of a landed staging entry's ready flag (early-fill engine)
__device__ __forceinline__ int fill_tag(int step, int layer) { return step * 256 + layer + 1; }
__device__ __forceinline__ void red_add_u64(long long *p, long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace m2c

// api.cu -- the C ABI of libm2c (include/m2c.h): validation, memory layout, stream/event
// orchestration, CUDA-graph capture of the decode step, NCCL (dlopen) for d_ff sharding.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "m2c_internal.cuh"

namespace m2c {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }
m2c_status fail(m2c_status st, const std::string &msg) {
    g_err = msg;
    return st;
}
m2c_status cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return M2C_ERR_CUDA;
}

size_t lru_smem_bytes(int P2, int maxcnt);

// ---- NCCL, loaded at run time (no link-time dependency) ----
typedef int ncclResult_t;
typedef void *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, int, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*errStr)(ncclResult_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

static NcclApi *load_nccl(const char *path) {
    static NcclApi api;
    if (api.h) return &api;
    const char *cands[] = {path, "libnccl.so.2", "libnccl.so"};
    for (const char *p : cands) {
        if (!p) continue;
        api.h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
    }
    if (!api.h) return nullptr;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(api.h, "ncclCommInitRank");
    api.allReduce = (decltype(api.allReduce))dlsym(api.h, "ncclAllReduce");
    api.commDestroy = (decltype(api.commDestroy))dlsym(api.h, "ncclCommDestroy");
    api.errStr = (decltype(api.errStr))dlsym(api.h, "ncclGetErrorString");
    api.allGather = (decltype(api.allGather))dlsym(api.h, "ncclAllGather");
    if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy) {
        dlclose(api.h);
        api.h = nullptr;
        return nullptr;
    }
    return &api;
}

// ---- per-layer memory layout (hbm_region / host_region) ----
struct Layout {
    size_t A = 0, B = 0, pool[3] = {0, 0, 0}, occ[3] = {0, 0, 0}, last[3] = {0, 0, 0},
           slot_of[3] = {0, 0, 0}, ord[3] = {0, 0, 0}, hbm = 0;
    size_t host_rec[3] = {0, 0, 0}, host = 0;
};
static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

static Layout layout_of(const m2c_model_desc &d, const m2c_cache_cfg &cfg) {
    Layout L;
    const int64_t F_r = d.d_ff / d.shard_count;
    const int bits[3] = {16, 8, 4};
    size_t off = 0;
    L.A = off;
    off += a256((size_t)d.pred_rank * d.d_model);
    L.B = off;
    off += a256((size_t)F_r * d.pred_rank);
    for (int t = 0; t < 3; t++) {
        const int64_t cap = cfg.mode == 0 ? F_r : cfg.cap_slots[t];
        L.pool[t] = off;
        off += a256((size_t)cap * m2c_record_bytes(bits[t], d.d_model));
    }
    if (cfg.mode != 0) {
        for (int t = 0; t < 3; t++) {
            L.occ[t] = off;
            off += a256(4 * (size_t)cfg.cap_slots[t]);
            L.last[t] = off;
            off += a256(4 * (size_t)cfg.cap_slots[t]);
            L.slot_of[t] = off;
            off += a256(4 * (size_t)F_r);
            L.ord[t] = off;
            off += a256(4 * (size_t)cfg.cap_slots[t]);
        }
        size_t h = 0;
        for (int t = 0; t < 3; t++) {
            L.host_rec[t] = h;
            h += a256((size_t)F_r * m2c_record_bytes(bits[t], d.d_model));
        }
        L.host = h;
    }
    L.hbm = off;
    return L;
}

static m2c_status check_desc(const m2c_model_desc *d) {
    if (!d) return fail(M2C_ERR_INVALID_ARG, "null model desc");
    if (d->d_model <= 0 || d->d_model % 256 || d->d_model > 8192)
        return fail(M2C_ERR_CONFIG, "d_model must be a positive multiple of 256, <= 8192");
    if (d->group != 128) return fail(M2C_ERR_CONFIG, "group must be 128 (R4)");
    if (d->pred_rank < 16 || d->pred_rank % 16 || d->pred_rank > 512 ||
        ((d->pred_rank / 16) & (d->pred_rank / 16 - 1)))
        return fail(M2C_ERR_CONFIG, "pred_rank must be 16 * 2^j <= 512");
    if (d->shard_count < 1 || d->shard_index < 0 || d->shard_index >= d->shard_count ||
        d->d_ff <= 0 || d->d_ff % d->shard_count)
        return fail(M2C_ERR_CONFIG, "bad d_ff / shard");
    if (d->d_ff / d->shard_count > (1 << 20)) return fail(M2C_ERR_CONFIG, "F_r too large");
    if (d->n_layers < 1) return fail(M2C_ERR_CONFIG, "n_layers < 1");
    if (d->act != 0 && d->act != 1) return fail(M2C_ERR_CONFIG, "act must be 0 (SiLU) or 1 (ReLU)");
    return M2C_OK;
}

static m2c_status check_plan(const m2c_tier_plan *p, int F_r) {
    if (!p) return fail(M2C_ERR_INVALID_ARG, "null plan");
    if (p->k < 0 || p->k > F_r || p->k_fp16 < 0 || p->k_int8 < 0 || p->k_int4 < 0 ||
        (int64_t)p->k_fp16 + p->k_int8 + p->k_int4 != p->k)
        return fail(M2C_ERR_CONFIG, "tier plan: need k16 + k8 + k4 == k <= F_r");
    return M2C_OK;
}

static bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// a device-side invariant violation of an earlier call (flag_error) makes the
// next host call return M2C_ERR_STATE.  Reads the pinned mirror only (no synchronisation);
// reporting clears it (the device word keeps the bits for m2c_stats).
static std::string err_bits_text(uint32_t err) {
    std::string m;
    if (err & 1) m += " non-finite input x;";
    if (err & 4) m += " decode grid-barrier timeout;";
    if (err & 8) m += " decode select count mismatch;";
    if (err & 16) m += " p2p exchange timeout (a peer rank is not running);";
    return m;
}
static m2c_status check_device_flag(m2c_ctx *c) {
    const uint32_t v = c && c->err_host ? *reinterpret_cast<volatile uint32_t *>(c->err_host) : 0u;
    if (!v) return M2C_OK;
    *reinterpret_cast<volatile uint32_t *>(c->err_host) = 0;
    return fail(M2C_ERR_STATE, "device flagged an invariant violation in an earlier call:" +
                                   err_bits_text(v & 0x7fffffffu));
}
#define M2C_CHECK_DEVICE_FLAG(c)                               \
    do {                                                       \
        m2c_status _s = check_device_flag(c);                  \
        if (_s != M2C_OK) return _s;                           \
    } while (0)

static int32_t *step_ptr(m2c_ctx *c) { return c->ws.counts + 15; }

// ---- the token: all layers on the compute stream (+ copy stream for LRU fills) ----
// profiling events per layer: 5 compute-stream marks (phase boundaries) + 2 around the miss
// fill on the copy stream
constexpr int kProfEv = 11;  // (early-fill engine: + 7 after the LRU update, 8 after the hit FFN,
                             // 9 after the miss queue, 10 after the requantisation)
static cudaError_t mark_copy(m2c_ctx *c, int l, int i) {
    if (c->prof_ev.empty()) return cudaSuccess;
    return cudaEventRecordWithFlags(c->prof_ev[kProfEv * l + 5 + i], c->copy, cudaEventRecordExternal);
}
static cudaError_t mark(m2c_ctx *c, int l, int i) {
    if (c->prof_ev.empty()) return cudaSuccess;
    return cudaEventRecordWithFlags(c->prof_ev[kProfEv * l + i], c->compute, cudaEventRecordExternal);
}

// the miss fill of layer l: from the in-memory host tier, or (NEXT-1) from the layer's DRAM
// frame of the SSD store -- the host blocks until the preloader has it resident
static cudaError_t enqueue_fill(m2c_ctx *c, int l, const m2c_tier_plan &p, int stage_par = -1) {
    const LayerState &L = c->layers[l];
    if (!c->store) return launch_fill(c, L, p, c->copy, stage_par);
    uint8_t *frame = store_acquire(c, l);
    if (!frame) return cudaErrorUnknown;  // I/O error (m2c_last_error is set by the caller)
    LayerState F = L;
    for (int t = 0; t < 3; t++) F.host_rec[t] = frame + L.host_off[t];
    cudaError_t e = launch_fill(c, F, p, c->copy);
    store_release(c, l, c->copy);
    return e;
}

// k_decode's P2/P3 (predictor + distributed exact select) and FFN share fit the kernel
static bool decode_select_ok(const m2c_ctx *c) { return decode_shape_ok(c); }

// the early-fill LRU engine: not with the NEXT-2 lookahead or a NEXT-1 store (their fills
// have their own sources); M2C_EARLY_FILL=0 disables it (A/B knob, results identical)
static bool early_fill_on(const m2c_ctx *c) {
    static const bool env_on = !(getenv("M2C_EARLY_FILL") && atoi(getenv("M2C_EARLY_FILL")) == 0);
    return env_on && c->early_fill && c->early_mem && !c->lookahead && !c->store;
}

// the miss FFN overlapped with the fill through per-record flags (early-fill engine);
// M2C_OVERLAP=0 disables it (A/B knob, results identical)
static bool overlap_on(const m2c_ctx *c) {
    static const bool env_on = !(getenv("M2C_OVERLAP") && atoi(getenv("M2C_OVERLAP")) == 0);
    (void)c;
    return env_on;
}

// GPU requantisation of INT misses from resident FP16 records (early-fill engine);
// M2C_REQUANT=0 disables it (A/B knob, results identical)
static bool requant_on(const m2c_ctx *c) {
    static const bool env_on = !(getenv("M2C_REQUANT") && atoi(getenv("M2C_REQUANT")) == 0);
    return env_on && c->requant;
}

static cudaError_t early_fill_alloc(m2c_ctx *c) {
    if (c->early_mem) return cudaSuccess;
    const m2c_tier_plan &p = c->plan;
    const int k = p.k > 0 ? p.k : 1;
    const int kt[3] = {p.k_fp16, p.k_int8, p.k_int4};
    size_t off = a256(4 * (16 + (size_t)k)) + 4 * a256(4 * (size_t)k), st_off[3];
    for (int t = 0; t < 3; t++) {
        st_off[t] = off;
        off += a256((size_t)(kt[t] > 0 ? kt[t] : 1) * c->nb[t]);
    }
    cudaError_t e = cudaMalloc(&c->early_mem, off);
    if (e) return e;
    uint8_t *b = static_cast<uint8_t *>(c->early_mem);
    c->mq = reinterpret_cast<int32_t *>(b);
    c->ident = reinterpret_cast<int32_t *>(b + a256(4 * (16 + (size_t)k)));
    c->mq_src = reinterpret_cast<int32_t *>(b + a256(4 * (16 + (size_t)k)) + a256(4 * (size_t)k));
    c->mq_job = reinterpret_cast<int32_t *>(b + a256(4 * (16 + (size_t)k)) + 2 * a256(4 * (size_t)k));
    c->mq_ready = reinterpret_cast<int32_t *>(b + a256(4 * (16 + (size_t)k)) + 3 * a256(4 * (size_t)k));
    for (int t = 0; t < 3; t++) c->mstage[t] = b + st_off[t];
    std::vector<int32_t> id(k, 0);
    for (int t = 0, seg = 0; t < 3; seg += kt[t], t++)
        for (int m = 0; m < kt[t]; m++) id[seg + m] = m;
    if ((e = cudaMemset(c->mq, 0, 4 * (16 + (size_t)k)))) return e;
    if ((e = cudaMemset(c->mq_ready, 0, 4 * (size_t)k))) return e;  // (no tag is 0)
    if ((e = cudaMemcpy(c->ident, id.data(), 4 * (size_t)k, cudaMemcpyHostToDevice))) return e;
    if ((e = cudaEventCreateWithFlags(&c->ev_q, cudaEventDisableTiming))) return e;
    if ((e = cudaEventCreateWithFlags(&c->ev_rq, cudaEventDisableTiming))) return e;
    if ((e = cudaStreamCreateWithFlags(&c->rq_stream, cudaStreamNonBlocking))) return e;
    return cudaEventCreateWithFlags(&c->ev_scat, cudaEventDisableTiming);
}

static cudaError_t enqueue_layer(m2c_ctx *c, int l, __half *x) {
    LayerState &L = c->layers[l];
    const m2c_tier_plan &p = c->plan;
    cudaStream_t st = c->compute;
    cudaError_t e;
    // resident: predictor (+ score histogram, + L2 prefetch of the previous token's records)
    // -> multi-CTA select writing this layer's tier lists -> FFN -> reduce (PDL-chained).
    // The lists of layer l persist to the next token as its prefetch hint.
    int32_t *lists = c->prev_ids + (size_t)l * (p.k > 0 ? p.k : 1);
    const bool prefetch = L.mode == 0 && c->use_fused;
    int32_t *ids = lists;  // this layer's tier lists (kept per layer: m2c_decode_lists)
    if ((e = mark(c, l, 0))) return e;
    if (c->trace_x && (e = cudaMemcpyAsync(c->trace_x + (size_t)l * c->desc.d_model, x, 2 * (size_t)c->desc.d_model,
                                           cudaMemcpyDeviceToDevice, st)))
        return e;
    if (L.mode != 0 && c->lookahead && !c->store && l + 1 < c->desc.n_layers) {
        // NEXT-2: predict layer l+1's selection from x_l first, and stage its would-be
        // misses on the staging stream (its own PCIe transfer, concurrent with this layer's)
        const LayerState &Ln = c->layers[l + 1];
        if ((e = launch_predict(c, Ln, x, c->ws.s, c->ghist, nullptr, st))) return e;
        if ((e = launch_select(c, c->ws.s, c->ghist, p, nullptr, nullptr, c->spec_ids, st))) return e;
        // the staging buffers of this parity were last read by layer l-1's fill (copy stream)
        if (l > 0 && (e = cudaStreamWaitEvent(st, c->ev_fill, 0))) return e;
        if ((e = launch_stage_plan(c, Ln, (l + 1) & 1, c->spec_ids, st))) return e;
        if ((e = cudaEventRecord(c->ev_stage, st))) return e;
        if ((e = cudaStreamWaitEvent(c->stage_stream, c->ev_stage, 0))) return e;
        if ((e = launch_stage_fill(c, Ln, (l + 1) & 1, c->stage_stream))) return e;
        if ((e = cudaEventRecord(c->ev_staged[(l + 1) & 1], c->stage_stream))) return e;
    }
    if (L.mode == 0 && c->comm && c->global_topk) {
        // NEXT-3: exact global top-k -- local candidates (top min(F_r, k) by (score desc,
        // global id asc)), an all-gather of the keys, the global cuts, this rank's share
        const m2c_tier_plan &g = c->gplan;
        const int n = g.k < c->F_r ? g.k : c->F_r;
        if (!c->nccl || !c->nccl->allGather) return cudaErrorNotSupported;  // NCCL without ncclAllGather
        const m2c_tier_plan pc{n, n, 0, 0};
        if ((e = launch_predict(c, L, x, c->ws.s, c->ghist, nullptr, st))) return e;
        if ((e = mark(c, l, 1))) return e;
        if ((e = launch_select(c, c->ws.s, c->ghist, pc, c->ws.slots, nullptr, c->ws.tier_ids, st))) return e;
        if ((e = launch_cand_keys(c, c->ws.s, c->ws.slots, n, c->gkeys, st))) return e;
        if (c->nccl->allGather(c->gkeys, c->gkeys + n, (size_t)n, 4 /*int64*/, c->comm, st) != 0)
            return cudaErrorUnknown;
        if ((e = launch_select_global(c, c->gkeys + n, n, g, c->gids, c->ws.counts, st))) return e;
        if ((e = mark(c, l, 2))) return e;
        if ((e = launch_ffn(c, L, x, c->gids, c->ws.counts, g, c->ws.partial, st))) return e;
        if ((e = mark(c, l, 3))) return e;
        if ((e = launch_reduce(c, c->G, c->ws.partial, x, c->ws.y32, nullptr, nullptr, nullptr, st))) return e;
        if (c->nccl->allReduce(c->ws.y32, c->ws.y32, (size_t)c->desc.d_model, 7 /*f32*/, 0 /*sum*/, c->comm, st) != 0)
            return cudaErrorUnknown;
        if ((e = launch_finalize(c, c->ws.y32, x, nullptr, x, st))) return e;
        if (c->trace_y && (e = cudaMemcpyAsync(c->trace_y + (size_t)l * c->desc.d_model, c->ws.y32,
                                               4 * (size_t)c->desc.d_model, cudaMemcpyDeviceToDevice, st)))
            return e;
        return mark(c, l, 4);
    }
    if (L.mode != 0 && c->use_fused && decode_select_ok(c)) {
        // the predictor + exact select of k_decode in one launch (its P2/P3 phases)
        if ((e = launch_decode(c, x, c->prof_ev.empty() ? nullptr : c->dec_prof, st, l, 1, nullptr,
                               nullptr, ids, l > 0 && c->h_prepared)))
            return e;
        c->h_prepared = false;
        // (rank order -> ascending ids per tier: the order the LRU update pairs misses in, R7;
        // the early-fill engine's k_missq sorts them itself)
        if (!early_fill_on(c) && (e = launch_sort_tiers(c, ids, p, st))) return e;
        if ((e = mark(c, l, 1))) return e;
        if ((e = mark(c, l, 2))) return e;
    } else {
        if ((e = launch_predict(c, L, x, c->ws.s, c->ghist, prefetch ? lists : nullptr, st))) return e;
        if ((e = mark(c, l, 1))) return e;
        if ((e = launch_select(c, c->ws.s, c->ghist, p, nullptr, nullptr, ids, st))) return e;
        if ((e = mark(c, l, 2))) return e;
    }
    int np = c->G;
    if (L.mode == 0) {
        e = launch_ffn(c, L, x, ids, c->ws.counts, p, c->ws.partial, st);
        if (e) return e;
    } else if (early_fill_on(c)) {
        // early fill: the misses (ids without a slot) are queued first and their host-tier
        // copies start into the staging area while k_lru chooses the victims; the miss FFN
        // reads the staging area; the copy stream then scatters the records into their slots
        // An INT8 / INT4 miss whose neuron is resident in the FP16 pool is filled by quantising
        // that record on the GPU (k_requant, the offline pack's function) instead of over PCIe
        const bool rq = requant_on(c);
        // (mq_src always written: -1 = a host copy; the fill and the miss FFN's waits read it)
        if ((e = launch_missq(c, L, ids, p, st, c->mq_src, decode_select_ok(c), rq))) return e;
        if ((e = mark(c, l, 9))) return e;
        if ((e = cudaEventRecord(c->ev_q, st))) return e;
        if ((e = cudaStreamWaitEvent(c->copy, c->ev_q, 0))) return e;
        if ((e = mark_copy(c, l, 0))) return e;
        const uint8_t *hsrc[3] = {L.host_rec[0], L.host_rec[1], L.host_rec[2]};
        const bool ovl = overlap_on(c);
        if ((e = launch_copy_recs(c, hsrc, c->mstage, p, c->mq, c->mq + 16, c->ident, c->copy,
                                  c->mq_src, ovl ? l : -1)))
            return e;
        // the requantisation on its own stream: k_lru and the hit FFN do not need it; the
        // scatter (it may overwrite an FP16 victim the requantisation reads) and the miss FFN do
        if (rq) {
            if ((e = cudaStreamWaitEvent(c->rq_stream, c->ev_q, 0))) return e;
            if ((e = launch_requant(c, L, p, c->rq_stream))) return e;
            if ((e = cudaEventRecord(c->ev_rq, c->rq_stream))) return e;
        }
        if ((e = mark(c, l, 10))) return e;
        if ((e = mark_copy(c, l, 1))) return e;
        if ((e = cudaEventRecord(c->ev_fill, c->copy))) return e;
        // the previous layer's scatter (copy stream) reads ws.counts[8..10] and ws.miss_items,
        // which this k_lru rewrites: join it first (it overlapped that layer's miss FFN, reduce
        // and this layer's select, so the wait is normally already satisfied)
        if (c->scat_pending && (e = cudaStreamWaitEvent(st, c->ev_scat, 0))) return e;
        e = launch_lru(c, L, step_ptr(c), ids, p, c->ws.slots, c->ws.hit_bits, nullptr, nullptr, st);
        if (e) return e;
        if ((e = mark(c, l, 7))) return e;
        if ((e = cudaEventRecord(c->ev_lookup, st))) return e;
        if ((e = cudaStreamWaitEvent(c->copy, c->ev_lookup, 0))) return e;
        if (rq && (e = cudaStreamWaitEvent(c->copy, c->ev_rq, 0))) return e;
        const uint8_t *ssrc[3] = {c->mstage[0], c->mstage[1], c->mstage[2]};
        uint8_t *pdst[3] = {L.pool[0], L.pool[1], L.pool[2]};
        if ((e = launch_copy_recs(c, ssrc, pdst, p, c->ws.counts, c->ident, c->ws.miss_items, c->copy)))
            return e;
        if ((e = cudaEventRecord(c->ev_scat, c->copy))) return e;
        c->scat_pending = true;
        e = launch_ffn(c, L, x, c->ws.hit_items, c->ws.counts + 4, p, c->ws.partial, st);
        if (e) return e;
        if ((e = mark(c, l, 8))) return e;
        // the miss FFN: with the overlap it starts now and takes each record as it lands
        // (k_fill's per-record flags); else after the whole fill
        if (!ovl && (e = cudaStreamWaitEvent(st, c->ev_fill, 0))) return e;
        if (rq && (e = cudaStreamWaitEvent(st, c->ev_rq, 0))) return e;
        LayerState Ls = L;
        for (int t = 0; t < 3; t++) Ls.pool[t] = c->mstage[t];
        e = launch_ffn(c, Ls, x, c->ident, c->mq + 8, p, c->ws.partial + (size_t)c->G * c->desc.d_model, st,
                       ovl ? l : -1);
        if (e) return e;
        np = 2 * c->G;
    } else {
        e = launch_lru(c, L, step_ptr(c), ids, p, c->ws.slots, c->ws.hit_bits, nullptr, nullptr, st);
        if (e) return e;
        if ((e = cudaEventRecord(c->ev_lookup, st))) return e;
        if ((e = cudaStreamWaitEvent(c->copy, c->ev_lookup, 0))) return e;
        // NEXT-2: layer l's records staged during layer l-1 (parity l & 1) fill device-side
        const bool la = c->lookahead && !c->store;
        if (la && l > 0 && (e = cudaStreamWaitEvent(c->copy, c->ev_staged[l & 1], 0))) return e;
        if ((e = mark_copy(c, l, 0))) return e;
        if ((e = enqueue_fill(c, l, p, la && l > 0 ? (l & 1) : -1))) return e;
        if ((e = mark_copy(c, l, 1))) return e;
        if (la && l > 0 && (e = launch_stage_clear(c, L, l & 1, c->copy))) return e;
        if ((e = cudaEventRecord(c->ev_fill, c->copy))) return e;
        e = launch_ffn(c, L, x, c->ws.hit_items, c->ws.counts + 4, p, c->ws.partial, st);
        if (e) return e;
        if ((e = cudaStreamWaitEvent(st, c->ev_fill, 0))) return e;
        e = launch_ffn(c, L, x, c->ws.miss_items, c->ws.counts + 8, p,
                       c->ws.partial + (size_t)c->G * c->desc.d_model, st);
        if (e) return e;
        np = 2 * c->G;
    }
    if ((e = mark(c, l, 3))) return e;
    if (c->comm) {  // (a communicator makes the collectives run, even for one rank)
        if ((e = launch_reduce(c, np, c->ws.partial, x, c->ws.y32, nullptr, nullptr, nullptr, st)))
            return e;
        int r = c->nccl->allReduce(c->ws.y32, c->ws.y32, (size_t)c->desc.d_model, 7 /*f32*/,
                                   0 /*sum*/, c->comm, st);
        if (r != 0) return cudaErrorUnknown;
        if ((e = launch_finalize(c, c->ws.y32, x, nullptr, x, st))) return e;
        if (c->trace_y && (e = cudaMemcpyAsync(c->trace_y + (size_t)l * c->desc.d_model, c->ws.y32,
                                               4 * (size_t)c->desc.d_model, cudaMemcpyDeviceToDevice, st)))
            return e;
    } else {
        float *ytr = c->trace_y ? c->trace_y + (size_t)l * c->desc.d_model : nullptr;
        // the next layer's select-only k_decode: its h (and a clear histogram) from this reduce
        const bool prep = l + 1 < c->desc.n_layers && c->layers[l + 1].mode != 0 && c->use_fused &&
                          decode_select_ok(c) && !c->lookahead && !c->store;
        if ((e = launch_reduce(c, np, c->ws.partial, x, ytr, nullptr, x, prep ? c->dec_hist : nullptr, st,
                               prep ? c->layers[l + 1].A : nullptr)))
            return e;
        c->h_prepared = prep;
    }
    return mark(c, l, 4);
}

// the persistent decode kernel covers a resident, unsharded stack whose scores fit in smem
static bool decode_fused(const m2c_ctx *c) {
    const int rps = (c->F_r + c->G - 1) / c->G;  // a CTA's own neurons: one pass of its threads
    (void)rps;
    if (!c->use_fused || (c->comm && !c->p2p) || !decode_shape_ok(c)) return false;
    for (const LayerState &L : c->layers)
        if (L.mode != 0) return false;
    return true;
}

// the layer-split engine: k_decode one layer per launch, the d_ff shards' partial y summed by
// one NCCL all-reduce between launches (the next launch adds it into x); resident stacks only
static bool decode_split(const m2c_ctx *c) {
    if (!c->use_fused || c->global_topk || (!c->comm && !c->force_split)) return false;
    const int rps = (c->F_r + c->G - 1) / c->G;
    (void)rps;
    if (!decode_shape_ok(c)) return false;
    for (const LayerState &L : c->layers)
        if (L.mode != 0) return false;
    return true;
}

static cudaError_t enqueue_token(m2c_ctx *c, __half *x) {
    const m2c_tier_plan &p = c->plan;
    c->last_token_fused = decode_fused(c) && !c->force_split;
    c->last_token_split = !c->last_token_fused && decode_split(c);
    if (c->last_token_fused)
        return launch_decode(c, x, c->prof_ev.empty() ? nullptr : c->dec_prof, c->compute);
    if (c->last_token_split) {
        unsigned long long *prof = c->prof_ev.empty() ? nullptr : c->dec_prof;
        cudaError_t e;
        const size_t d = c->desc.d_model;
        for (int l = 0; l < c->desc.n_layers; l++) {
            if ((e = launch_decode(c, x, prof, c->compute, l, 1, l > 0 ? c->ws.y32 : nullptr, c->ws.y32))) return e;
            if (c->comm && c->nccl->allReduce(c->ws.y32, c->ws.y32, d, 7 /*f32*/,
                                                    0 /*sum*/, c->comm, c->compute) != 0)
                return cudaErrorUnknown;
            if (c->trace_y && (e = cudaMemcpyAsync(c->trace_y + l * d, c->ws.y32, 4 * d,
                                                   cudaMemcpyDeviceToDevice, c->compute)))
                return e;
        }
        if ((e = launch_finalize(c, c->ws.y32, x, nullptr, x, c->compute))) return e;
        if (c->trace_x)
            return cudaMemcpyAsync(c->trace_x + c->desc.n_layers * d, x, 2 * d, cudaMemcpyDeviceToDevice, c->compute);
        return cudaSuccess;
    }
    cudaError_t e = launch_set_counts(c->ws.counts, p.k_fp16, p.k_int8, p.k_int4, c->compute);
    c->launch_counter++;
    if (e) return e;
    bool early = false;
    for (int l = 0; l < c->desc.n_layers; l++) {
        if ((e = enqueue_layer(c, l, x))) return e;
        early |= c->layers[l].mode != 0 && early_fill_on(c);
    }
    if (c->trace_x &&
        (e = cudaMemcpyAsync(c->trace_x + (size_t)c->desc.n_layers * c->desc.d_model, x,
                             2 * (size_t)c->desc.d_model, cudaMemcpyDeviceToDevice, c->compute)))
        return e;
    if (early) {
        c->scat_pending = false;
        return cudaStreamWaitEvent(c->compute, c->ev_scat, 0);  // join the last scatter
    }
    return cudaSuccess;
}

}  // namespace m2c

using namespace m2c;

extern "C" {

const char *m2c_last_error(void) { return g_err.c_str(); }
int32_t m2c_abi_version(void) { return M2C_ABI_VERSION; }

int64_t m2c_record_bytes(int32_t bits, int32_t d) {
    if (d <= 0 || d % 128) return -1;
    const int64_t G = d / 128;
    int64_t raw;
    if (bits == 16) raw = 6LL * d;
    else if (bits == 8) raw = 3LL * d + 9 * G;
    else if (bits == 4) raw = 3LL * d / 2 + 9 * G;
    else return -1;
    return (raw + 15) / 16 * 16;
}

m2c_status m2c_tier_plan_make(int32_t F_r, int32_t pct, int32_t a16, int32_t a8, int32_t den,
                              m2c_tier_plan *out) {
    if (!out || F_r < 0 || pct < 0 || pct > 100 || den <= 0 || a16 < 0 || a8 < 0 || a16 + a8 > den)
        return fail(M2C_ERR_INVALID_ARG, "tier_plan_make: bad arguments");
    const int64_t k = (int64_t)F_r * pct / 100;
    const int64_t k16 = k * a16 / den, k8 = k * a8 / den;
    out->k = (int32_t)k;
    out->k_fp16 = (int32_t)k16;
    out->k_int8 = (int32_t)k8;
    out->k_int4 = (int32_t)(k - k16 - k8);
    return M2C_OK;
}

m2c_status m2c_cache_cfg_capped(const m2c_model_desc *desc, const m2c_tier_plan *plan,
                                int32_t num, int32_t den, int32_t mode, m2c_cache_cfg *out) {
    m2c_status st = check_desc(desc);
    if (st) return st;
    const int F_r = desc->d_ff / desc->shard_count;
    if ((st = check_plan(plan, F_r))) return st;
    if (!out || num <= 0 || den <= 0 || (mode != 1 && mode != 2))
        return fail(M2C_ERR_INVALID_ARG, "cache_cfg_capped: bad arguments");
    const int kt[3] = {plan->k_fp16, plan->k_int8, plan->k_int4};
    const int bits[3] = {16, 8, 4};
    out->mode = mode;
    if (mode == 2) {  // ATU: exactly the active set
        for (int t = 0; t < 3; t++) out->cap_slots[t] = kt[t];
        return M2C_OK;
    }
    double act_bytes = 0;
    for (int t = 0; t < 3; t++) act_bytes += (double)kt[t] * m2c_record_bytes(bits[t], desc->d_model);
    const double budget = (double)num / den * 6.0 * desc->d_model * F_r;
    const double M = act_bytes > 0 ? budget / act_bytes : 0;
    for (int t = 0; t < 3; t++) {
        double c = std::floor(M * kt[t]);
        if (c > F_r) c = F_r;
        out->cap_slots[t] = (int32_t)c;
    }
    return M2C_OK;
}

m2c_status m2c_layer_footprint(const m2c_model_desc *desc, const m2c_cache_cfg *cfg,
                               size_t *hbm, size_t *host) {
    m2c_status st = check_desc(desc);
    if (st) return st;
    if (!cfg || cfg->mode < 0 || cfg->mode > 2) return fail(M2C_ERR_INVALID_ARG, "bad cache cfg");
    const Layout L = layout_of(*desc, *cfg);
    if (hbm) *hbm = L.hbm;
    if (host) *host = L.host;
    return M2C_OK;
}

m2c_status m2c_create(const m2c_model_desc *desc, int32_t device, m2c_stream_t compute,
                      m2c_stream_t copy, const m2c_tier_plan *plan, m2c_ctx **out) {
    m2c_status st = check_desc(desc);
    if (st) return st;
    const int F_r = desc->d_ff / desc->shard_count;
    if ((st = check_plan(plan, F_r))) return st;
    if (!out) return fail(M2C_ERR_INVALID_ARG, "null out");
    int ndev = 0;
    M2C_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(M2C_ERR_INVALID_ARG, "bad device");
    M2C_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    M2C_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(M2C_ERR_CONFIG, "libm2c is built for sm_100a (B200) only");
    m2c_ctx *c = new m2c_ctx();
    c->desc = *desc;
    c->F_r = F_r;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->G = prop.multiProcessorCount;
    c->compute = reinterpret_cast<cudaStream_t>(compute);
    c->copy = reinterpret_cast<cudaStream_t>(copy);
    c->plan = *plan;
    const int bits[3] = {16, 8, 4};
    for (int t = 0; t < 3; t++) c->nb[t] = m2c_record_bytes(bits[t], desc->d_model);
    c->layers.resize(desc->n_layers);
    // workspace
    const int d = desc->d_model, r = desc->pred_rank;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += a256(bytes);
        return o;
    };
    const size_t o_h = take(8 * (size_t)kHStride * r), o_s = take(4 * (size_t)F_r),
                 o_ids = take(4 * (size_t)F_r), o_tof = take((size_t)F_r),
                 o_slots = take(4 * (size_t)F_r), o_bits = take(4 * ((size_t)F_r / 32 + 2)),
                 o_hit = take(4 * (size_t)F_r), o_miss = take(4 * (size_t)F_r),
                 o_mid = take(4 * (size_t)F_r), o_cnt = take(4 * 16),
                 o_part = take(4 * (size_t)2 * c->G * d), o_y = take(4 * (size_t)d),
                 o_x = take(2 * (size_t)d), o_stats = take(8 * 16), o_err = take(16),
                 o_hist = take(4 * 2 * 4096), o_sst = take(8 * (size_t)select_blocks(F_r)),
                 o_sdone = take(4), o_sepoch = take(4), o_bflags = take(4 * (size_t)c->G),
                 o_bepoch = take(4), o_dlay = take(decode_layer_table_bytes(desc->n_layers)),
                 o_dprof = take(8 * (size_t)kDecodeStamps * c->G * desc->n_layers),
                 o_binsh = take(4 * (size_t)desc->n_layers), o_sabs = take(8 * (size_t)c->G),
                 o_hb = take(8 * 2 * (size_t)kHStride * r),
                 o_bucket = take(decode_bucket_bytes()), o_sdump = take(4 * (size_t)F_r),
                 o_dhist = take(decode_hist_bytes()),
                 o_prev = take(4 * (size_t)desc->n_layers * (plan->k > 0 ? plan->k : 1));
    // score histogram geometry: |s| <= 127^2 r, bins of 2^sh over [0, 2 smax] (4096 bins)
    c->sel_smax = 16129 * desc->pred_rank;
    {
        int bits = 0;
        while ((1LL << bits) <= 2LL * c->sel_smax) bits++;
        c->sel_sh = bits > 12 ? bits - 12 : 0;
    }
    cudaError_t e = cudaMalloc(&c->ws_mem, off);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaMalloc(workspace)");
    }
    c->ws_bytes = off;
    uint8_t *b = static_cast<uint8_t *>(c->ws_mem);
    c->ws.h = (long long *)(b + o_h);
    c->ws.s = (int32_t *)(b + o_s);
    c->ws.tier_ids = (int32_t *)(b + o_ids);
    c->ws.tier_of = (int8_t *)(b + o_tof);
    c->ws.slots = (int32_t *)(b + o_slots);
    c->ws.hit_bits = (uint32_t *)(b + o_bits);
    c->ws.hit_items = (int32_t *)(b + o_hit);
    c->ws.miss_items = (int32_t *)(b + o_miss);
    c->ws.miss_ids = (int32_t *)(b + o_mid);
    c->ws.counts = (int32_t *)(b + o_cnt);
    c->ws.partial = (float *)(b + o_part);
    c->ws.y32 = (float *)(b + o_y);
    c->ws.xbuf = (__half *)(b + o_x);
    c->ws.stats = (unsigned long long *)(b + o_stats);
    c->ws.err = (uint32_t *)(b + o_err);
    c->ghist = (int *)(b + o_hist);
    c->prev_ids = (int32_t *)(b + o_prev);
    c->sel_status = (unsigned long long *)(b + o_sst);
    c->sel_done = (int *)(b + o_sdone);
    c->sel_epoch = (int *)(b + o_sepoch);
    c->bar_flags = (unsigned *)(b + o_bflags);
    c->bar_epoch = (unsigned *)(b + o_bepoch);
    c->dec_layers = b + o_dlay;
    c->dec_prof = (unsigned long long *)(b + o_dprof);
    c->dec_bin_sh = (int *)(b + o_binsh);
    c->dec_sabs = (unsigned *)(b + o_sabs);
    c->dec_hb = (long long *)(b + o_hb);
    c->dec_bucket = (unsigned long long *)(b + o_bucket);
    c->dec_sdump = (int *)(b + o_sdump);
    c->dec_hist = (int *)(b + o_dhist);
    e = cudaMemset(c->ws_mem, 0, off);
    if (e == cudaSuccess) {  // k_decode's first token: a histogram scale that covers |s| <= smax
        int sh0 = 0;
        while ((c->sel_smax >> sh0) >= 2048) sh0++;
        std::vector<int> v(desc->n_layers, sh0);
        e = cudaMemcpy(c->dec_bin_sh, v.data(), 4 * v.size(), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess)  // no previous selection yet: -1 disables the prefetch hint
        e = cudaMemset(c->prev_ids, 0xff, 4 * (size_t)desc->n_layers * (plan->k > 0 ? plan->k : 1));
    // kernel attributes (max dynamic smem) are per device: set once per device
    static uint64_t attrs_done = 0;  // bit = device index (< 64)
    if (e == cudaSuccess && !(device < 64 && ((attrs_done >> device) & 1))) {
        e = init_select_attrs();
        if (e == cudaSuccess) e = init_cache_attrs();
        if (e == cudaSuccess) e = init_ffn_attrs();
        if (e == cudaSuccess) e = init_decode_attrs();
        if (e == cudaSuccess && device < 64) attrs_done |= 1ull << device;
    }
    // the device error word's pinned host mirror (flag_error): the next host call sees it
    if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void **>(&c->err_host), 4, cudaHostAllocMapped);
    if (e == cudaSuccess) {
        *c->err_host = 0;
        void *dptr = nullptr;
        e = cudaHostGetDevicePointer(&dptr, c->err_host, 0);
        if (e == cudaSuccess) e = cudaMemcpy(c->ws.err + 2, &dptr, sizeof(dptr), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fill_api, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_lookup, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fill, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_stage, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        m2c_destroy(c);
        return cuda_fail(e, "m2c_create");
    }
    *out = c;
    return M2C_OK;
}

m2c_status m2c_destroy(m2c_ctx *c) {
    if (!c) return M2C_OK;
    if (c->store) {
        cudaStreamSynchronize(c->copy);
        store_close(c);
    }
    if (c->graph) cudaGraphExecDestroy(c->graph);
    for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
    if (c->comm && c->nccl) c->nccl->commDestroy(c->comm);
    if (c->ev_lookup) cudaEventDestroy(c->ev_lookup);
    if (c->ev_fill) cudaEventDestroy(c->ev_fill);
    if (c->ev_stage) cudaEventDestroy(c->ev_stage);
    if (c->gkeys) cudaFree(c->gkeys);
    if (c->stage_mem) {
        cudaStreamSynchronize(c->stage_stream);
        cudaStreamDestroy(c->stage_stream);
        for (int p = 0; p < 2; p++) cudaEventDestroy(c->ev_staged[p]);
        cudaFree(c->stage_mem);
    }
    if (c->early_mem) {
        cudaStreamSynchronize(c->copy);
        cudaFree(c->early_mem);
    }
    if (c->ev_q) cudaEventDestroy(c->ev_q);
    if (c->ev_rq) cudaEventDestroy(c->ev_rq);
    if (c->rq_stream) {
        cudaStreamSynchronize(c->rq_stream);
        cudaStreamDestroy(c->rq_stream);
    }
    if (c->ev_scat) cudaEventDestroy(c->ev_scat);
    for (void *p : c->p2p_opened) cudaIpcCloseMemHandle(p);
    if (c->p2p_tabs) cudaFree(c->p2p_tabs);
    if (c->p2p_mem) cudaFree(c->p2p_mem);
    if (c->ws_mem) cudaFree(c->ws_mem);
    if (c->err_host) cudaFreeHost(c->err_host);
    if (c->ev_fill_api) cudaEventDestroy(c->ev_fill_api);
    delete c;
    return M2C_OK;
}

m2c_status m2c_quant_pack(int32_t d, int32_t bits, const void *g, const void *u, const void *dn,
                          int64_t n0, int64_t n1, void *out, m2c_stream_t stream) {
    if (d <= 0 || d % 128) return fail(M2C_ERR_INVALID_ARG, "quant_pack: d % 128 != 0");
    if (bits != 16 && bits != 8 && bits != 4) return fail(M2C_ERR_INVALID_ARG, "quant_pack: bits");
    if (!g || !u || !dn || !out || n0 < 0 || n1 < n0)
        return fail(M2C_ERR_INVALID_ARG, "quant_pack: null pointer or bad range");
    if (!al16(g) || !al16(u) || !al16(dn) || !al16(out))
        return fail(M2C_ERR_INVALID_ARG, "quant_pack: pointers must be 16-B aligned");
    M2C_CUDA(launch_pack(d, bits, (const __half *)g, (const __half *)u, (const __half *)dn, n0, n1,
                         (uint8_t *)out, reinterpret_cast<cudaStream_t>(stream)));
    return M2C_OK;
}

m2c_status m2c_load_layer(m2c_ctx *c, int32_t layer, const void *g, const void *u, const void *dn,
                          const int8_t *A, const int8_t *B, const m2c_cache_cfg *cfg,
                          void *hbm_region, void *host_region) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !cfg || !g || !u || !dn || !A || !B || !hbm_region)
        return fail(M2C_ERR_INVALID_ARG, "load_layer: null argument");
    if (layer < 0 || layer >= c->desc.n_layers) return fail(M2C_ERR_INVALID_ARG, "bad layer");
    if (cfg->mode < 0 || cfg->mode > 2) return fail(M2C_ERR_INVALID_ARG, "bad cache mode");
    if ((reinterpret_cast<uintptr_t>(hbm_region) & 255) ||
        (host_region && (reinterpret_cast<uintptr_t>(host_region) & 255)))
        return fail(M2C_ERR_INVALID_ARG, "regions must be 256-B aligned");
    if (!al16(g) || !al16(u) || !al16(dn)) return fail(M2C_ERR_INVALID_ARG, "masters not 16-B aligned");
    const int kt[3] = {c->plan.k_fp16, c->plan.k_int8, c->plan.k_int4};
    if (cfg->mode != 0) {
        if (!host_region) return fail(M2C_ERR_INVALID_ARG, "LRU/ATU needs a pinned host region");
        for (int t = 0; t < 3; t++)
            if (cfg->cap_slots[t] < kt[t] || cfg->cap_slots[t] > kMaxPoolSlots ||
                cfg->cap_slots[t] > c->F_r)
                return fail(M2C_ERR_CAPACITY, "pool capacity must be in [k_t, min(F_r, 8192)]");
    }
    const Layout Lo = layout_of(c->desc, *cfg);
    cudaStream_t st = c->compute;
    const int d = c->desc.d_model, r = c->desc.pred_rank, F_r = c->F_r;
    uint8_t *hb = static_cast<uint8_t *>(hbm_region);
    uint8_t *hh = static_cast<uint8_t *>(host_region);
    LayerState &L = c->layers[layer];
    L = LayerState();
    L.mode = cfg->mode;
    L.A = (const int8_t *)(hb + Lo.A);
    L.B = (const int8_t *)(hb + Lo.B);
    // A arrives row-major [r][d]; it is stored transposed (A^T [d][r], R2 / k_pred.cu).  The
    // FFN partial-sum workspace (8 G d >= r d bytes) stages the transpose.
    M2C_CUDA(cudaMemcpyAsync(c->ws.partial, A, (size_t)r * d, cudaMemcpyDefault, st));
    M2C_CUDA(launch_transpose_i8(r, d, (const int8_t *)c->ws.partial, (int8_t *)(hb + Lo.A), st));
    M2C_CUDA(cudaMemcpyAsync(hb + Lo.B, B, (size_t)F_r * r, cudaMemcpyDefault, st));
    const int bits[3] = {16, 8, 4};
    const __half *G = (const __half *)g, *U = (const __half *)u, *D = (const __half *)dn;
    for (int t = 0; t < 3; t++) {
        L.pool[t] = hb + Lo.pool[t];
        L.cap[t] = cfg->mode == 0 ? F_r : cfg->cap_slots[t];
        if (cfg->mode == 0) {
            M2C_CUDA(launch_pack(d, bits[t], G, U, D, 0, F_r, L.pool[t], st));
        } else {
            // pack chunk-wise into the (cold) pool memory as scratch, then copy to the host tier
            uint8_t *dst = hh + Lo.host_rec[t];
            const int64_t chunk = L.cap[t];
            for (int64_t n0 = 0; n0 < F_r; n0 += chunk) {
                const int64_t n1 = n0 + chunk < F_r ? n0 + chunk : F_r;
                M2C_CUDA(launch_pack(d, bits[t], G, U, D, n0, n1, L.pool[t], st));
                M2C_CUDA(cudaMemcpyAsync(dst + n0 * c->nb[t], L.pool[t], (n1 - n0) * c->nb[t],
                                         cudaMemcpyDefault, st));
            }
            L.host_rec[t] = dst;
            L.host_base = hh;
            L.host_off[t] = Lo.host_rec[t];
            L.host_bytes = Lo.host;
            L.occupant[t] = (int32_t *)(hb + Lo.occ[t]);
            L.last[t] = (int32_t *)(hb + Lo.last[t]);
            L.slot_of[t] = (int32_t *)(hb + Lo.slot_of[t]);
            L.ord[t] = (int32_t *)(hb + Lo.ord[t]);
            M2C_CUDA(launch_iota(L.ord[t], L.cap[t], st));  // all last_use = -1: slot order
            M2C_CUDA(launch_fill_i32(L.occupant[t], -1, L.cap[t], st));
            M2C_CUDA(launch_fill_i32(L.last[t], -1, L.cap[t], st));
            M2C_CUDA(launch_fill_i32(L.slot_of[t], -1, F_r, st));
        }
    }
    M2C_CUDA(cudaStreamSynchronize(st));
    L.loaded = true;
    c->dec_table_dirty = true;
    if (c->graph) {  // topology may have changed
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return M2C_OK;
}

m2c_status m2c_predict_rank(m2c_ctx *c, int32_t layer, const void *x, const m2c_tier_plan *plan,
                            int32_t *rank_list, int8_t *tier_of, int32_t *tier_ids,
                            int32_t *scores) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !x || !plan || (!tier_ids && plan->k > 0))
        return fail(M2C_ERR_INVALID_ARG, "predict_rank: null argument");
    if (layer < 0 || layer >= c->desc.n_layers || !c->layers[layer].loaded)
        return fail(M2C_ERR_STATE, "predict_rank: layer not loaded");
    m2c_status st = check_plan(plan, c->F_r);
    if (st) return st;
    if (!al16(x)) return fail(M2C_ERR_INVALID_ARG, "x must be 16-B aligned");
    if (rank_list && plan->k > 16384)
        return fail(M2C_ERR_CAPACITY, "rank_list: k too large for the on-chip sort (<= 16384)");
    int32_t *s = scores ? scores : c->ws.s;
    // the select kernel consumes and clears the score histogram the predictor builds
    M2C_CUDA(launch_predict(c, c->layers[layer], (const __half *)x, s, c->ghist, nullptr, c->compute));
    M2C_CUDA(launch_select(c, s, c->ghist, *plan, rank_list, tier_of, tier_ids, c->compute));
    return M2C_OK;
}

m2c_status m2c_cache_lookup_fill(m2c_ctx *c, int32_t layer, int64_t step, const int32_t *tier_ids,
                                 const m2c_tier_plan *plan, int32_t *slots, uint32_t *hit_bitmap,
                                 int32_t *miss_log, int32_t *evict_log, int32_t *counts,
                                 m2c_event_t fill_done) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !plan || !hit_bitmap || ((!tier_ids || !slots) && plan->k > 0))
        return fail(M2C_ERR_INVALID_ARG, "cache_lookup_fill: null argument");
    if (layer < 0 || layer >= c->desc.n_layers || !c->layers[layer].loaded)
        return fail(M2C_ERR_STATE, "cache_lookup_fill: layer not loaded");
    m2c_status st = check_plan(plan, c->F_r);
    if (st) return st;
    LayerState &L = c->layers[layer];
    if (step <= L.last_step || step > INT32_MAX - 2 || step < 0)
        return fail(M2C_ERR_STATE, "cache_lookup_fill: step must strictly increase (0..2^31-3)");
    cudaStream_t cs = c->compute;
    const size_t nbits = sizeof(uint32_t) * ((plan->k + 31) / 32);  // the documented size exactly
    if (L.mode == 0) {  // resident: identity, all hits
        M2C_CUDA(cudaMemcpyAsync(slots, tier_ids, 4 * (size_t)plan->k, cudaMemcpyDeviceToDevice, cs));
        if (nbits) M2C_CUDA(cudaMemsetAsync(hit_bitmap, 0, nbits, cs));
        if (plan->k) M2C_CUDA(cudaMemsetAsync(hit_bitmap, 0xff, 4 * (size_t)(plan->k / 32), cs));
        if (plan->k % 32) {
            const uint32_t tail = (1u << (plan->k % 32)) - 1;
            M2C_CUDA(cudaMemcpyAsync(hit_bitmap + plan->k / 32, &tail, 4, cudaMemcpyHostToDevice, cs));
        }
        if (counts) M2C_CUDA(cudaMemsetAsync(counts, 0, 6 * sizeof(int32_t), cs));
        M2C_CUDA(launch_set_counts(c->ws.counts + 4, plan->k_fp16, plan->k_int8, plan->k_int4, cs));
        M2C_CUDA(launch_set_counts(c->ws.counts + 8, 0, 0, 0, cs));
        M2C_CUDA(cudaMemcpyAsync(c->ws.hit_items, tier_ids, 4 * (size_t)plan->k, cudaMemcpyDeviceToDevice, cs));
        if (fill_done) M2C_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(fill_done), cs));
    } else {
        for (int t = 0; t < 3; t++) {
            const int kt = t == 0 ? plan->k_fp16 : (t == 1 ? plan->k_int8 : plan->k_int4);
            if (kt > L.cap[t]) return fail(M2C_ERR_CAPACITY, "k_t exceeds the pool capacity");
        }
        const int32_t st32 = (int32_t)step;
        M2C_CUDA(cudaMemcpyAsync(step_ptr(c), &st32, 4, cudaMemcpyHostToDevice, cs));
        // an earlier lookup's fill (copy stream) may still read the workspace miss lists that
        // this k_lru rewrites
        if (c->fill_pending) M2C_CUDA(cudaStreamWaitEvent(cs, c->ev_fill_api, 0));
        M2C_CUDA(launch_lru(c, L, step_ptr(c), tier_ids, *plan, slots, hit_bitmap, miss_log, evict_log, cs));
        if (counts) {
            M2C_CUDA(cudaMemcpyAsync(counts, c->ws.counts + 8, 12, cudaMemcpyDeviceToDevice, cs));
            M2C_CUDA(cudaMemcpyAsync(counts + 3, c->ws.counts + 12, 12, cudaMemcpyDeviceToDevice, cs));
        }
        M2C_CUDA(cudaEventRecord(c->ev_lookup, cs));
        M2C_CUDA(cudaStreamWaitEvent(c->copy, c->ev_lookup, 0));
        M2C_CUDA(enqueue_fill(c, layer, *plan));
        M2C_CUDA(cudaEventRecord(c->ev_fill_api, c->copy));
        c->fill_pending = true;
        if (fill_done) M2C_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(fill_done), c->copy));
    }
    c->ws_lists_layer = layer;  // the hit / miss lists m2c_sparse_ffn_forward will read
    L.last_step = step;
    return M2C_OK;
}

m2c_status m2c_sparse_ffn_forward(m2c_ctx *c, int32_t layer, const void *x, const int32_t *tier_ids,
                                  const int32_t *slots, const uint32_t *hit_bitmap,
                                  const m2c_tier_plan *plan, m2c_event_t fill_done,
                                  float *y_partial, void *y) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !x || !plan || (!tier_ids && plan->k > 0))
        return fail(M2C_ERR_INVALID_ARG, "sparse_ffn_forward: null argument");
    if (layer < 0 || layer >= c->desc.n_layers || !c->layers[layer].loaded)
        return fail(M2C_ERR_STATE, "sparse_ffn_forward: layer not loaded");
    m2c_status st = check_plan(plan, c->F_r);
    if (st) return st;
    if (!al16(x)) return fail(M2C_ERR_INVALID_ARG, "x must be 16-B aligned");
    LayerState &L = c->layers[layer];
    if (L.mode != 0 && !hit_bitmap)
        return fail(M2C_ERR_STATE, "LRU/ATU layer: pass the lookup's slots and hit_bitmap");
    if (hit_bitmap && c->ws_lists_layer != layer)
        return fail(M2C_ERR_STATE, "sparse_ffn_forward: the context's hit / miss lists belong to "
                                   "another layer -- call m2c_cache_lookup_fill for this layer "
                                   "right before its FFN (m2c.h)");
    cudaStream_t cs = c->compute;
    const __half *xh = (const __half *)x;
    const int d = c->desc.d_model;
    int np = c->G;
    M2C_CUDA(launch_set_counts(c->ws.counts, plan->k_fp16, plan->k_int8, plan->k_int4, cs));
    if (!hit_bitmap) {
        M2C_CUDA(launch_ffn(c, L, xh, slots ? slots : tier_ids, c->ws.counts, *plan, c->ws.partial, cs));
    } else {
        // hits first, then wait for the fills, then the misses (R11)
        M2C_CUDA(launch_ffn(c, L, xh, c->ws.hit_items, c->ws.counts + 4, *plan, c->ws.partial, cs));
        if (fill_done) M2C_CUDA(cudaStreamWaitEvent(cs, reinterpret_cast<cudaEvent_t>(fill_done), 0));
        M2C_CUDA(launch_ffn(c, L, xh, c->ws.miss_items, c->ws.counts + 8, *plan,
                            c->ws.partial + (size_t)c->G * d, cs));
        np = 2 * c->G;
    }
    if (c->comm) {
        M2C_CUDA(launch_reduce(c, np, c->ws.partial, xh, c->ws.y32, nullptr, nullptr, nullptr, cs));
        if (y_partial)
            M2C_CUDA(cudaMemcpyAsync(y_partial, c->ws.y32, 4 * (size_t)d, cudaMemcpyDeviceToDevice, cs));
        if (y) {
            int r = c->nccl->allReduce(c->ws.y32, c->ws.y32, (size_t)d, 7, 0, c->comm, cs);
            if (r) return fail(M2C_ERR_NCCL, c->nccl->errStr ? c->nccl->errStr(r) : "ncclAllReduce");
            M2C_CUDA(launch_finalize(c, c->ws.y32, xh, (__half *)y, nullptr, cs));
        }
    } else {
        M2C_CUDA(launch_reduce(c, np, c->ws.partial, xh, y_partial, (__half *)y, nullptr, nullptr, cs));
    }
    return M2C_OK;
}

m2c_status m2c_nccl_unique_id(const char *lib, void *id_out) {
    if (!id_out) return fail(M2C_ERR_INVALID_ARG, "null id");
    NcclApi *api = load_nccl(lib);
    if (!api) return fail(M2C_ERR_NCCL, "cannot dlopen libnccl.so.2");
    ncclUniqueId id;
    int r = api->getUniqueId(&id);
    if (r) return fail(M2C_ERR_NCCL, api->errStr ? api->errStr(r) : "ncclGetUniqueId");
    memcpy(id_out, &id, sizeof(id));
    return M2C_OK;
}

m2c_status m2c_comm_init(m2c_ctx *c, int32_t nranks, int32_t rank, const void *uid, const char *lib) {
    if (!c || !uid) return fail(M2C_ERR_INVALID_ARG, "comm_init: null argument");
    if (nranks != c->desc.shard_count || rank != c->desc.shard_index)
        return fail(M2C_ERR_CONFIG, "comm_init: nranks/rank must equal shard_count/shard_index");
    // (nranks == 1 is allowed: a one-rank communicator makes the sharded engines run their
    // collectives as identities -- the single-GPU test of the NCCL wiring)
    NcclApi *api = load_nccl(lib);
    if (!api) return fail(M2C_ERR_NCCL, "cannot dlopen libnccl.so.2");
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    M2C_CUDA(cudaSetDevice(c->device));
    ncclComm_t comm = nullptr;
    int r = api->commInitRank(&comm, nranks, id, rank);
    if (r) return fail(M2C_ERR_NCCL, api->errStr ? api->errStr(r) : "ncclCommInitRank");
    c->nccl = api;
    c->comm = comm;
    c->nranks = nranks;
    c->rank = rank;
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return M2C_OK;
}

m2c_status m2c_set_grid(m2c_ctx *c, int32_t ctas) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    if (ctas < 1 || ctas > c->num_sms) return fail(M2C_ERR_INVALID_ARG, "set_grid: 1 <= ctas <= SM count");
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    // k_decode's grid barrier waits for (epoch + n) * G arrivals on one counter: a new G needs
    // a fresh counter (after every launch of the old grid has drained)
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    M2C_CUDA(cudaMemset(c->bar_flags, 0, 4 * (size_t)c->num_sms));
    M2C_CUDA(cudaMemset(c->bar_epoch, 0, 4));
    c->G = ctas;
    return M2C_OK;
}

// §8(e) exchange buffer of this rank: [2 (round parity)][P][d] u64 (flag << 32 | f32) | u32 rounds
static size_t p2p_rounds_off(const m2c_ctx *c) { return 16 * (size_t)c->desc.shard_count * c->desc.d_model; }

m2c_status m2c_p2p_buffer(m2c_ctx *c, uint64_t *dev_ptr_out, void *ipc_handle_out) {
    if (!c || !dev_ptr_out) return fail(M2C_ERR_INVALID_ARG, "p2p_buffer: null argument");
    if (c->desc.shard_count < 2) return fail(M2C_ERR_CONFIG, "p2p_buffer: needs shard_count >= 2");
    M2C_CUDA(cudaSetDevice(c->device));
    if (!c->p2p_mem) {
        c->p2p_bytes = p2p_rounds_off(c) + 256;
        M2C_CUDA(cudaMalloc(&c->p2p_mem, c->p2p_bytes));
        M2C_CUDA(cudaMemset(c->p2p_mem, 0, c->p2p_bytes));  // flags and rounds start at 0
        M2C_CUDA(cudaDeviceSynchronize());
    }
    *dev_ptr_out = (uint64_t)(uintptr_t)c->p2p_mem;
    if (ipc_handle_out) {
        cudaIpcMemHandle_t h;
        M2C_CUDA(cudaIpcGetMemHandle(&h, c->p2p_mem));
        memcpy(ipc_handle_out, &h, sizeof(h));
    }
    return M2C_OK;
}

m2c_status m2c_p2p_connect(m2c_ctx *c, int32_t nranks, const uint64_t *dev_ptrs, const void *ipc_handles) {
    if (!c || (!dev_ptrs && !ipc_handles)) return fail(M2C_ERR_INVALID_ARG, "p2p_connect: null argument");
    if (nranks != c->desc.shard_count || nranks < 2)
        return fail(M2C_ERR_CONFIG, "p2p_connect: nranks must equal shard_count (>= 2)");
    if (!c->p2p_mem) return fail(M2C_ERR_STATE, "p2p_connect: call m2c_p2p_buffer first");
    if (c->p2p) return fail(M2C_ERR_STATE, "p2p_connect: already connected");
    M2C_CUDA(cudaSetDevice(c->device));
    std::vector<uint8_t *> base(nranks);
    for (int q = 0; q < nranks; q++) {
        if (q == c->desc.shard_index) {
            base[q] = static_cast<uint8_t *>(c->p2p_mem);
        } else if (ipc_handles) {
            cudaIpcMemHandle_t h;
            memcpy(&h, static_cast<const uint8_t *>(ipc_handles) + (size_t)q * sizeof(h), sizeof(h));
            void *ptr = nullptr;
            M2C_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            c->p2p_opened.push_back(ptr);
            base[q] = static_cast<uint8_t *>(ptr);
        } else {
            base[q] = reinterpret_cast<uint8_t *>((uintptr_t)dev_ptrs[q]);
        }
    }
    M2C_CUDA(cudaMalloc(&c->p2p_tabs, sizeof(void *) * nranks));
    M2C_CUDA(cudaMemcpy(c->p2p_tabs, base.data(), sizeof(void *) * nranks, cudaMemcpyHostToDevice));
    c->p2p_xtab = static_cast<unsigned long long *const *>(c->p2p_tabs);
    c->p2p_rounds = reinterpret_cast<unsigned *>(base[c->desc.shard_index] + p2p_rounds_off(c));
    c->p2p = true;
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return M2C_OK;
}

m2c_status m2c_set_graph(m2c_ctx *c, int32_t enable) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    c->use_graph = enable != 0;
    return M2C_OK;
}

m2c_status m2c_set_fused(m2c_ctx *c, int32_t enable) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    c->use_fused = enable != 0;
    c->force_split = enable == 2;
    return M2C_OK;
}

m2c_status m2c_decode_step(m2c_ctx *c, void *x_inout, int64_t step) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !x_inout) return fail(M2C_ERR_INVALID_ARG, "decode_step: null argument");
    if (!al16(x_inout)) return fail(M2C_ERR_INVALID_ARG, "x must be 16-B aligned");
    bool any_lru = false;
    for (int l = 0; l < c->desc.n_layers; l++) {
        LayerState &L = c->layers[l];
        if (!L.loaded) return fail(M2C_ERR_STATE, "decode_step: a layer is not loaded");
        if (L.mode != 0) {
            any_lru = true;
            if (step <= L.last_step || step < 0 || step > INT32_MAX - 2)
                return fail(M2C_ERR_STATE, "decode_step: step must strictly increase");
        }
    }
    if (c->p2p && !c->comm && !(decode_fused(c) && !c->force_split))
        return fail(M2C_ERR_CONFIG, "decode_step: the p2p exchange runs only in the whole-token "
                                    "kernel and this stack/grid does not fit it (no communicator "
                                    "for the other engines)");
    cudaStream_t cs = c->compute;
    if (any_lru && !c->early_mem) M2C_CUDA(early_fill_alloc(c));
    if (any_lru) {
        const int32_t st32 = (int32_t)step;  // pageable source: staged before return
        M2C_CUDA(cudaMemcpyAsync(step_ptr(c), &st32, 4, cudaMemcpyHostToDevice, cs));
    }
    __half *x = static_cast<__half *>(x_inout);
    if (c->fill_pending) {  // a per-call lookup's fill may still read the workspace miss lists
        M2C_CUDA(cudaStreamWaitEvent(cs, c->ev_fill_api, 0));
        c->fill_pending = false;
    }
    if (c->dec_table_dirty) {  // pool / predictor pointers of every layer for k_decode
        M2C_CUDA(cudaStreamSynchronize(cs));
        M2C_CUDA(decode_write_layer_table(c, c->dec_layers));
        c->dec_table_dirty = false;
    }
    if (c->use_graph && !c->store) {  // (a store's frames change per token: eager)
        if (c->graph && c->graph_x != x_inout) {
            cudaGraphExecDestroy(c->graph);
            c->graph = nullptr;
        }
        if (!c->graph) {
            const int64_t before = c->launch_counter;
            cudaGraph_t g = nullptr;
            M2C_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = enqueue_token(c, x);
            cudaError_t e2 = cudaStreamEndCapture(cs, &g);
            if (e != cudaSuccess) {
                if (g) cudaGraphDestroy(g);
                return cuda_fail(e, "decode_step capture");
            }
            if (e2 != cudaSuccess) return cuda_fail(e2, "cudaStreamEndCapture");
            e = cudaGraphInstantiate(&c->graph, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
            c->graph_x = x_inout;
            c->kernels_per_token = c->launch_counter - before;
        }
        M2C_CUDA(cudaGraphLaunch(c->graph, cs));
    } else {
        const int64_t before = c->launch_counter;
        M2C_CUDA(enqueue_token(c, x));
        c->kernels_per_token = c->launch_counter - before;
    }
    for (int l = 0; l < c->desc.n_layers; l++)
        if (c->layers[l].mode != 0) c->layers[l].last_step = step;
    c->decoded = true;
    c->ws_lists_layer = -1;  // the engine reused the workspace lists
    return M2C_OK;
}

m2c_status m2c_decode_lists(m2c_ctx *c, int32_t layer, int32_t *tier_ids_out) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !tier_ids_out) return fail(M2C_ERR_INVALID_ARG, "decode_lists: null argument");
    if (layer < 0 || layer >= c->desc.n_layers) return fail(M2C_ERR_INVALID_ARG, "bad layer");
    if (!c->decoded) return fail(M2C_ERR_STATE, "decode_lists: no decode step yet");
    const m2c_tier_plan &p = c->plan;
    if (p.k_fp16 > sort_tiers_max() || p.k_int8 > sort_tiers_max() || p.k_int4 > sort_tiers_max())
        return fail(M2C_ERR_CAPACITY, "decode_lists: a tier has more than 32768 entries");
    const int k = p.k;
    if (k > 0) {
        // the engines keep each layer's selection in rank order (k_decode) or ascending per
        // tier (chain); the API returns three ascending segments
        M2C_CUDA(cudaMemcpyAsync(tier_ids_out, c->prev_ids + (size_t)layer * k, 4 * (size_t)k,
                                 cudaMemcpyDeviceToDevice, c->compute));
        M2C_CUDA(launch_sort_tiers(c, tier_ids_out, p, c->compute));
    }
    return M2C_OK;
}

m2c_status m2c_set_trace(m2c_ctx *c, void *x_trace, float *y_trace) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    c->trace_x = static_cast<__half *>(x_trace);
    c->trace_y = y_trace;
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return M2C_OK;
}

m2c_status m2c_cache_state(m2c_ctx *c, int32_t layer, int32_t tier, int32_t *occupant_out,
                           int32_t *last_out, int32_t *cap_out) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !cap_out) return fail(M2C_ERR_INVALID_ARG, "cache_state: null argument");
    if (layer < 0 || layer >= c->desc.n_layers || tier < 0 || tier > 2)
        return fail(M2C_ERR_INVALID_ARG, "cache_state: bad layer / tier");
    const LayerState &L = c->layers[layer];
    if (!L.loaded || L.mode == 0) return fail(M2C_ERR_STATE, "cache_state: not an LRU/ATU layer");
    *cap_out = L.cap[tier];
    const size_t b = 4 * (size_t)L.cap[tier];
    if (occupant_out)
        M2C_CUDA(cudaMemcpyAsync(occupant_out, L.occupant[tier], b, cudaMemcpyDeviceToDevice, c->compute));
    if (last_out) M2C_CUDA(cudaMemcpyAsync(last_out, L.last[tier], b, cudaMemcpyDeviceToDevice, c->compute));
    return M2C_OK;
}

m2c_status m2c_profile(m2c_ctx *c, int32_t enable) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
    c->prof_ev.clear();
    if (enable) {
        c->prof_ev.resize(kProfEv * (size_t)c->desc.n_layers);
        for (auto &e : c->prof_ev) M2C_CUDA(cudaEventCreate(&e));
    }
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return M2C_OK;
}

m2c_status m2c_profile_read(m2c_ctx *c, float *ms, int32_t *ffn_launches) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !ms) return fail(M2C_ERR_INVALID_ARG, "null argument");
    if (c->prof_ev.empty()) return fail(M2C_ERR_STATE, "profiling not enabled");
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    if (c->last_token_fused || c->last_token_split) {  // in-kernel per-CTA stamps (ns): see k_decode.cu
        const int L = c->desc.n_layers, G = c->G, S = kDecodeStamps;
        std::vector<unsigned long long> t((size_t)S * G * L);
        M2C_CUDA(cudaMemcpy(t.data(), c->dec_prof, 8 * t.size(), cudaMemcpyDeviceToHost));
        auto mx = [&](int l, int i) {
            unsigned long long v = 0;
            for (int g = 0; g < G; g++) v = std::max(v, t[((size_t)l * G + g) * S + i]);
            return v;
        };
        auto mn = [&](int l, int i) {
            unsigned long long v = ~0ull;
            for (int g = 0; g < G; g++) v = std::min(v, t[((size_t)l * G + g) * S + i]);
            return v;
        };
        for (int l = 0; l < L; l++) {
            const unsigned long long s0 = mn(l, 0), s4 = mx(l, 4), s5 = mx(l, 5), s7 = mx(l, 7);
            const unsigned long long nx = l + 1 < L ? mn(l + 1, 0) : mx(l, 9);
            ms[4 * l + 0] = (float)((double)(s4 - s0) * 1e-6);
            ms[4 * l + 1] = (float)((double)(s5 - s4) * 1e-6);
            ms[4 * l + 2] = (float)((double)(s7 - s5) * 1e-6);
            ms[4 * l + 3] = (float)((double)(nx - s7) * 1e-6);
        }
        if (ffn_launches) *ffn_launches = 0;
        return M2C_OK;
    }
    for (int l = 0; l < c->desc.n_layers; l++)
        for (int i = 0; i < 4; i++)
            M2C_CUDA(cudaEventElapsedTime(&ms[4 * l + i], c->prof_ev[kProfEv * l + i],
                                          c->prof_ev[kProfEv * l + i + 1]));
    if (ffn_launches) *ffn_launches = c->layers[0].mode == 0 ? 1 : 2;
    return M2C_OK;
}

m2c_status m2c_profile_fill(m2c_ctx *c, float *ms) {
    if (!c || !ms) return fail(M2C_ERR_INVALID_ARG, "null argument");
    if (c->prof_ev.empty()) return fail(M2C_ERR_STATE, "profiling not enabled");
    if (c->last_token_fused || c->last_token_split) return fail(M2C_ERR_STATE, "no fills in the last step");
    M2C_CUDA(cudaStreamSynchronize(c->copy));
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    for (int l = 0; l < c->desc.n_layers; l++) {
        ms[l] = 0.f;
        if (c->layers[l].mode == 0) continue;
        M2C_CUDA(cudaEventElapsedTime(&ms[l], c->prof_ev[kProfEv * l + 5], c->prof_ev[kProfEv * l + 6]));
    }
    return M2C_OK;
}

m2c_status m2c_profile_events(m2c_ctx *c, float *ms, int64_t cap, int64_t *n_out) {
    if (!c || !n_out) return fail(M2C_ERR_INVALID_ARG, "null argument");
    const int64_t n = (int64_t)kProfEv * c->desc.n_layers;
    *n_out = n;
    if (!ms) return M2C_OK;
    if (cap < n) return fail(M2C_ERR_INVALID_ARG, "profile_events: buffer too small");
    if (c->prof_ev.empty()) return fail(M2C_ERR_STATE, "profiling not enabled");
    if (c->last_token_fused || c->last_token_split)
        return fail(M2C_ERR_STATE, "profile_events: the last step was one k_decode launch (use m2c_profile_stamps)");
    M2C_CUDA(cudaStreamSynchronize(c->copy));
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    for (int l = 0; l < c->desc.n_layers; l++)
        for (int i = 0; i < kProfEv; i++) {
            float v = -1.f;  // (a mark the layer's engine did not record)
            if (i < 5 || (c->layers[l].mode != 0 && (i < 7 || early_fill_on(c))))  // (10: requant on)
                if (cudaEventElapsedTime(&v, c->prof_ev[0], c->prof_ev[kProfEv * l + i]) != cudaSuccess) v = -1.f;
            ms[kProfEv * l + i] = v;
        }
    cudaGetLastError();  // (an unrecorded mark leaves a sticky-free error)
    return M2C_OK;
}

m2c_status m2c_profile_stamps(m2c_ctx *c, uint64_t *out, int64_t cap, int64_t *n_out) {
    if (!c || !n_out) return fail(M2C_ERR_INVALID_ARG, "null argument");
    const int64_t n = (int64_t)kDecodeStamps * c->G * c->desc.n_layers;
    *n_out = n;
    if (!out) return M2C_OK;
    if (cap < n) return fail(M2C_ERR_INVALID_ARG, "profile_stamps: buffer too small");
    if (c->prof_ev.empty() || !(c->last_token_fused || c->last_token_split || decode_select_ok(c)))
        return fail(M2C_ERR_STATE, "profile_stamps: profiling off or last token not on k_decode");
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    M2C_CUDA(cudaMemcpy(out, c->dec_prof, 8 * (size_t)n, cudaMemcpyDeviceToHost));
    return M2C_OK;
}

m2c_status m2c_predict_candidates(m2c_ctx *c, int32_t layer, const void *x, int32_t n_cand,
                                  int64_t *keys_out) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !x || !keys_out) return fail(M2C_ERR_INVALID_ARG, "predict_candidates: null argument");
    if (layer < 0 || layer >= c->desc.n_layers || !c->layers[layer].loaded)
        return fail(M2C_ERR_STATE, "predict_candidates: layer not loaded");
    if (n_cand < 0 || n_cand > c->F_r || n_cand > 16384)
        return fail(M2C_ERR_CONFIG, "predict_candidates: need 0 <= n_cand <= min(F_r, 16384)");
    if (!al16(x)) return fail(M2C_ERR_INVALID_ARG, "x must be 16-B aligned");
    m2c_tier_plan p{n_cand, n_cand, 0, 0};
    M2C_CUDA(launch_predict(c, c->layers[layer], (const __half *)x, c->ws.s, c->ghist, nullptr, c->compute));
    M2C_CUDA(launch_select(c, c->ws.s, c->ghist, p, c->ws.slots /*rank order*/, nullptr, c->ws.tier_ids,
                           c->compute));
    M2C_CUDA(launch_cand_keys(c, c->ws.s, c->ws.slots, n_cand, reinterpret_cast<long long *>(keys_out), c->compute));
    return M2C_OK;
}

m2c_status m2c_select_global(m2c_ctx *c, const int64_t *keys_all, int32_t n_cand,
                             const m2c_tier_plan *global_plan, int32_t *tier_ids_out, int32_t *counts_out) {
    M2C_CHECK_DEVICE_FLAG(c);
    if (!c || !keys_all || !global_plan || !tier_ids_out || !counts_out)
        return fail(M2C_ERR_INVALID_ARG, "select_global: null argument");
    const int P = c->desc.shard_count;
    if (P > 32) return fail(M2C_ERR_CONFIG, "select_global: at most 32 ranks");
    const int64_t F = (int64_t)c->F_r * P;
    m2c_status st = check_plan(global_plan, (int32_t)(F < INT32_MAX ? F : INT32_MAX));
    if (st) return st;
    if (n_cand < (global_plan->k < c->F_r ? global_plan->k : c->F_r))
        return fail(M2C_ERR_CONFIG, "select_global: n_cand < min(F_r, k): the union would not be exact");
    if (8 * (size_t)P * n_cand > 200 * 1024)
        return fail(M2C_ERR_CAPACITY, "select_global: P x n_cand candidates exceed the on-chip buffer");
    M2C_CUDA(launch_select_global(c, reinterpret_cast<const long long *>(keys_all), n_cand, *global_plan,
                                  tier_ids_out, counts_out, c->compute));
    return M2C_OK;
}

m2c_status m2c_set_global_topk(m2c_ctx *c, const m2c_tier_plan *global_plan) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    if (!global_plan) {
        c->global_topk = false;
        return M2C_OK;
    }
    const int P = c->desc.shard_count;
    m2c_status st = check_plan(global_plan, c->F_r * P);
    if (st) return st;
    const int n = global_plan->k < c->F_r ? global_plan->k : c->F_r;
    if (8 * (size_t)P * n > 200 * 1024 || P > 32 || n > 16384)
        return fail(M2C_ERR_CAPACITY, "global top-k: P x min(F_r, k) candidates exceed the on-chip buffer");
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    if (c->gkeys) cudaFree(c->gkeys);
    c->gkeys = nullptr;
    // keys: own [n] + gathered [P][n]; then this layer's global lists [k_global]
    const size_t kb = 8 * (size_t)(P + 1) * (n > 0 ? n : 1), lb = 4 * (size_t)(global_plan->k > 0 ? global_plan->k : 1);
    M2C_CUDA(cudaMalloc(&c->gkeys, kb + lb));
    c->gids = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(c->gkeys) + kb);
    c->gplan = *global_plan;
    c->global_topk = true;
    return M2C_OK;
}

m2c_status m2c_set_lookahead(m2c_ctx *c, int32_t enable) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    M2C_CUDA(cudaStreamSynchronize(c->copy));
    if (c->stage_stream) M2C_CUDA(cudaStreamSynchronize(c->stage_stream));
    if (enable && !c->stage_mem) {
        const int F = c->F_r, k = c->plan.k > 0 ? c->plan.k : 1;
        const int kt[3] = {c->plan.k_fp16, c->plan.k_int8, c->plan.k_int4};
        size_t off = 0;
        auto take = [&](size_t b) {
            const size_t o = off;
            off += a256(b);
            return o;
        };
        size_t o_of[2], o_buf[2][3], o_sid[2];
        for (int p = 0; p < 2; p++) {
            o_of[p] = take(4 * 3 * (size_t)F);
            for (int t = 0; t < 3; t++) o_buf[p][t] = take((size_t)(kt[t] > 0 ? kt[t] : 1) * c->nb[t]);
            o_sid[p] = take(4 * (size_t)k);
        }
        const size_t o_spec = take(4 * (size_t)k);
        M2C_CUDA(cudaMalloc(&c->stage_mem, off));
        uint8_t *b = static_cast<uint8_t *>(c->stage_mem);
        for (int p = 0; p < 2; p++) {
            c->stage_of[p] = (int32_t *)(b + o_of[p]);
            for (int t = 0; t < 3; t++) c->stage_buf[p][t] = b + o_buf[p][t];
            c->stage_sid[p] = (int32_t *)(b + o_sid[p]);
            M2C_CUDA(cudaMemset(c->stage_of[p], 0xff, 4 * 3 * (size_t)F));  // -1: nothing staged
        }
        c->spec_ids = (int32_t *)(b + o_spec);
        M2C_CUDA(cudaStreamCreateWithFlags(&c->stage_stream, cudaStreamNonBlocking));
        for (int p = 0; p < 2; p++) M2C_CUDA(cudaEventCreateWithFlags(&c->ev_staged[p], cudaEventDisableTiming));
    }
    c->lookahead = enable != 0;
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return M2C_OK;
}

m2c_status m2c_requant_stats(m2c_ctx *c, int64_t *requant_fills, int32_t reset) {
    if (!c || !requant_fills) return fail(M2C_ERR_INVALID_ARG, "null argument");
    M2C_CHECK_DEVICE_FLAG(c);
    unsigned long long v[3] = {0, 0, 0};
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    M2C_CUDA(cudaMemcpy(v, c->ws.stats + 8, sizeof(v), cudaMemcpyDeviceToHost));
    for (int t = 0; t < 3; t++) requant_fills[t] = (int64_t)v[t];
    if (reset) M2C_CUDA(cudaMemset(c->ws.stats + 8, 0, sizeof(v)));
    return M2C_OK;
}

m2c_status m2c_set_requant(m2c_ctx *c, int32_t enable) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    c->requant = enable != 0;
    if (c->graph) {  // (the captured decode graph bakes the engine's launches in)
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return M2C_OK;
}

m2c_status m2c_lookahead_stats(m2c_ctx *c, int64_t *staged_fills, int32_t reset) {
    if (!c || !staged_fills) return fail(M2C_ERR_INVALID_ARG, "null argument");
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    M2C_CUDA(cudaStreamSynchronize(c->copy));
    if (c->stage_stream) M2C_CUDA(cudaStreamSynchronize(c->stage_stream));
    unsigned long long v = 0;
    M2C_CUDA(cudaMemcpy(&v, c->ws.stats + 6, 8, cudaMemcpyDeviceToHost));
    *staged_fills = (int64_t)v;
    if (reset) M2C_CUDA(cudaMemset(c->ws.stats + 6, 0, 8));
    return M2C_OK;
}

m2c_status m2c_store_write(m2c_ctx *c, const char *path) {
    if (!c || !path) return fail(M2C_ERR_INVALID_ARG, "store_write: null argument");
    M2C_CUDA(cudaDeviceSynchronize());
    return store_write(c, path, c->layers.empty() ? 0 : c->layers[0].host_bytes);
}

m2c_status m2c_store_attach(m2c_ctx *c, const char *path, int32_t n_fixed, int32_t n_dynamic,
                            int32_t lookahead, void *frames, size_t frames_bytes) {
    if (!c || !path || !frames) return fail(M2C_ERR_INVALID_ARG, "store_attach: null argument");
    if (c->store) return fail(M2C_ERR_STATE, "store_attach: a store is attached");
    const int L = c->desc.n_layers;
    if (n_fixed < 0 || n_dynamic < 0 || n_fixed > L || (n_fixed < L && n_dynamic < 1) || lookahead < 0)
        return fail(M2C_ERR_CONFIG, "store_attach: need 0 <= n_fixed <= L, n_dynamic >= 1 unless all layers are fixed");
    for (const LayerState &ls : c->layers)
        if (!ls.loaded || ls.mode == 0) return fail(M2C_ERR_STATE, "store_attach: all layers must be loaded in LRU/ATU mode");
    M2C_CUDA(cudaDeviceSynchronize());
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return store_open(c, path, n_fixed, n_dynamic, lookahead, frames, frames_bytes, c->layers[0].host_bytes);
}

m2c_status m2c_store_detach(m2c_ctx *c) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    if (!c->store) return M2C_OK;
    M2C_CUDA(cudaDeviceSynchronize());
    store_close(c);
    return M2C_OK;
}

m2c_status m2c_store_stats(m2c_ctx *c, int64_t *bytes_read, int64_t *layer_loads, double *io_seconds,
                           double *stall_seconds) {
    if (!c || !bytes_read || !layer_loads || !io_seconds || !stall_seconds)
        return fail(M2C_ERR_INVALID_ARG, "store_stats: null argument");
    if (!c->store) return fail(M2C_ERR_STATE, "store_stats: no store attached");
    store_stats(c, bytes_read, layer_loads, io_seconds, stall_seconds);
    return M2C_OK;
}

size_t m2c_store_frame_bytes(const m2c_model_desc *desc, const m2c_cache_cfg *cfg) {
    if (!desc || !cfg || cfg->mode == 0) return 0;
    const size_t h = layout_of(*desc, *cfg).host;
    return (h + 4095) / 4096 * 4096;
}

m2c_status m2c_stats(m2c_ctx *c, int64_t *kpt, int64_t hits[3], int64_t misses[3], int32_t reset) {
    if (!c) return fail(M2C_ERR_INVALID_ARG, "null ctx");
    if (kpt) *kpt = c->kernels_per_token;
    unsigned long long h[6] = {0, 0, 0, 0, 0, 0};
    M2C_CUDA(cudaStreamSynchronize(c->compute));
    M2C_CUDA(cudaMemcpy(h, c->ws.stats, sizeof(h), cudaMemcpyDeviceToHost));
    uint32_t err = 0;
    M2C_CUDA(cudaMemcpy(&err, c->ws.err, 4, cudaMemcpyDeviceToHost));
    for (int t = 0; t < 3; t++) {
        if (hits) hits[t] = (int64_t)h[t];
        if (misses) misses[t] = (int64_t)h[3 + t];
    }
    if (reset) M2C_CUDA(cudaMemset(c->ws.stats, 0, sizeof(h)));
    if (c->err_host) *reinterpret_cast<volatile uint32_t *>(c->err_host) = 0;
    if (err) {
        cudaMemset(c->ws.err, 0, 4);
        return fail(M2C_ERR_STATE, "device flagged:" + err_bits_text(err));
    }
    return M2C_OK;
}

}  // extern "C"

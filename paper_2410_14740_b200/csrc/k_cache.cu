// k_cache.cu -- a4/a5: the per-(layer, tier) neuron cache in HBM and the miss fills.
//
// Paper: one isolated, contiguous cache unit per layer whose memory is used in place by the
// computation; "a neuron-level mixed-precision LRU cache in HBM";
// misses loaded "asynchronously from DRAM to HBM to overlap the HBM cache miss with the GPU
// computation" on "dedicated CUDA streams".  The paper keeps the bookkeeping on
// the host; we keep it on the device because host-driven cache management costs a
// device->host round trip per layer ("GPU kernels are launched by CPUs").
// Policy details (the paper is silent): DESIGN.md R7 -- step-granular timestamps, victims =
// smallest (last_use, slot) with last_use < t, misses in ascending id paired with victims in
// that order; a tier change is a miss in the new tier's pool (R9).
#include <cstdlib>

#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int NT = 1024;
constexpr int NW = NT / 32;

struct LruArgs {
    int32_t *occ[3];
    int32_t *last[3];
    int32_t *slot_of[3];
    int32_t *ord[3];  // slots sorted by (last_use, slot): the LRU order, maintained in place
    int cap[3];
    int seg[3];
    int cnt[3];
};

// exclusive block scan of one int per thread
__device__ __forceinline__ int block_scan1(int v, int *tot, int *sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < NW) ? sm[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) sm[lane] = w;
    }
    __syncthreads();
    const int r = (warp ? sm[warp - 1] : 0) + x - v;
    *tot = sm[NW - 1];
    __syncthreads();
    return r;
}

// One CTA per tier pool.  The victims are the nm smallest (last_use, slot) among slots with
// last_use < t (R7).  Instead of sorting every step, the pool keeps its slots in that order
// (ord): after this step's hits are refreshed, the victims are the first nm non-hit entries of
// ord, and the new order is [the other non-hit entries, in order] ++ [hits and victims -- all
// now stamped t -- by slot].  O(C) with four block scans.
__global__ void __launch_bounds__(NT, 1)
    k_lru(LruArgs a, const int32_t *__restrict__ step_ptr, const int32_t *__restrict__ tier_ids, int32_t *__restrict__ slots,
          uint32_t *__restrict__ hit_bits, int32_t *__restrict__ hit_items,
          int32_t *__restrict__ miss_items, int32_t *__restrict__ miss_ids,
          int32_t *__restrict__ miss_log, int32_t *__restrict__ evict_log,
          int32_t *__restrict__ counts, unsigned long long *__restrict__ stats, int P2) {
    extern __shared__ __align__(16) uint8_t smraw[];
    // smem: new order [C] | victims [C] | miss positions [cnt] | the LRU order [C] | the tier's
    // ids [cnt] | their slots [cnt] | slot bitmaps hit, tail [C/32].  Every global array is read
    // once, coalesced, into shared memory up front: three dependent round trips in all (the
    // list + order, the list's slots, the victims' occupants), whatever the L2 latency while
    // the concurrent miss fill loads the memory system (round 2: ~10 before)
    int32_t *nord = reinterpret_cast<int32_t *>(smraw);
    int32_t *vict = nord + P2;
    int32_t *mpos = vict + P2;
    int32_t *sord = mpos + P2;
    int32_t *sR = sord + P2;
    int32_t *ssl = sR + P2;
    uint32_t *hmask = reinterpret_cast<uint32_t *>(ssl + P2);
    uint32_t *tmask = hmask + P2 / 32;
    __shared__ int scan_sm[NW];
    const int tau = blockIdx.x;
    const int n = a.cnt[tau], seg = a.seg[tau], C = a.cap[tau];
    for (int i = threadIdx.x; i < P2 / 32; i += NT) hmask[i] = tmask[i] = 0u;
    griddep_wait();
    const int t = *step_ptr;
    int32_t *occ = a.occ[tau], *last = a.last[tau], *slot_of = a.slot_of[tau], *ord = a.ord[tau];
    const int32_t *R = tier_ids + seg;
    for (int i = threadIdx.x; i < n; i += NT) sR[i] = R[i];
    for (int q = threadIdx.x; q < C; q += NT) sord[q] = ord[q];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) ssl[i] = slot_of[sR[i]];
    __syncthreads();

    // 1. hits: refresh their timestamp (a hit never moves slot)
    const int CH = (n + NT - 1) / NT;
    const int i0 = min(n, (int)threadIdx.x * CH), i1 = min(n, i0 + CH);
    int nh = 0;
    for (int i = i0; i < i1; i++) {
        const int sl = ssl[i];
        if (sl >= 0) {
            last[sl] = t;
            slots[seg + i] = sl;
            atomicOr(&hit_bits[(seg + i) >> 5], 1u << ((seg + i) & 31));
            atomicOr(&hmask[sl >> 5], 1u << (sl & 31));
            nh++;
        }
    }
    int tot_h;
    int hpos = block_scan1(nh, &tot_h, scan_sm);  // (a barrier: hmask complete)
    int mp = i0 - hpos;  // misses before this chunk = i0 - hits before it
    for (int i = i0; i < i1; i++) {
        const int sl = ssl[i];
        if (sl >= 0) hit_items[seg + hpos++] = sl;
        else mpos[mp++] = i;
    }
    const int nm = n - tot_h;
    // 2. victims: the first nm non-hit entries of the LRU order
    const int OC = (C + NT - 1) / NT;
    const int o0 = min(C, (int)threadIdx.x * OC), o1 = min(C, o0 + OC);
    int nk = 0;
    for (int q = o0; q < o1; q++) {
        const int sl = sord[q];
        nk += !((hmask[sl >> 5] >> (sl & 31)) & 1u);
    }
    int tot_k;
    int kpos = block_scan1(nk, &tot_k, scan_sm);  // non-hit rank of this thread's first entry
    for (int q = o0; q < o1; q++) {
        const int sl = sord[q];
        if ((hmask[sl >> 5] >> (sl & 31)) & 1u) continue;
        if (kpos < nm) {
            M2C_CHECK(sl >= 0 && sl < C);
            vict[kpos] = sl;
            atomicOr(&tmask[sl >> 5], 1u << (sl & 31));
        } else {
            nord[kpos - nm] = sl;  // kept, order preserved
        }
        kpos++;
    }
    __syncthreads();
    // 3. the tail: hits and victims by slot
    const int front = tot_k - nm;
    int nt = 0;
    for (int sl = o0; sl < o1; sl++)
        nt += ((hmask[sl >> 5] | tmask[sl >> 5]) >> (sl & 31)) & 1u;
    int tot_t;
    int tpos = block_scan1(nt, &tot_t, scan_sm) + front;
    for (int sl = o0; sl < o1; sl++)
        if (((hmask[sl >> 5] | tmask[sl >> 5]) >> (sl & 31)) & 1u) nord[tpos++] = sl;
    __syncthreads();
    for (int q = threadIdx.x; q < C; q += NT) ord[q] = nord[q];
    // 4. install misses[m] in victim[m]; evictions compacted in miss order
    const int MC = (nm + NT - 1) / NT;
    const int m0 = min(nm, (int)threadIdx.x * MC), m1 = min(nm, m0 + MC);
    int ne = 0;
    for (int m = m0; m < m1; m++) {
        const int o = occ[vict[m]];
        sord[m] = o;  // (the order was written out: its smem copy holds the victims' occupants)
        ne += o >= 0;
    }
    int tot_e;
    int epos = block_scan1(ne, &tot_e, scan_sm);
    M2C_CHECK(tot_k >= nm && nm <= C);  // enough non-hit slots to take every miss
    for (int m = m0; m < m1; m++) {
        const int i = mpos[m];
        const int id = sR[i];
        const int sl = vict[m];
        M2C_CHECK(i >= 0 && i < n && id >= 0 && sl >= 0 && sl < C);
        const int old = sord[m];
        if (old >= 0) {
            slot_of[old] = -1;
            if (evict_log) {
                evict_log[2 * (seg + epos)] = old;
                evict_log[2 * (seg + epos) + 1] = sl;
            }
            epos++;
        }
        occ[sl] = id;
        slot_of[id] = sl;
        last[sl] = t;
        slots[seg + i] = sl;
        miss_items[seg + m] = sl;
        miss_ids[seg + m] = id;
        if (miss_log) {
            miss_log[2 * (seg + m)] = id;
            miss_log[2 * (seg + m) + 1] = sl;
        }
    }
    if (threadIdx.x == 0) {
        counts[4 + tau] = tot_h;
        counts[8 + tau] = nm;
        counts[12 + tau] = tot_e;
        atomicAdd(&stats[tau], (unsigned long long)tot_h);
        atomicAdd(&stats[3 + tau], (unsigned long long)nm);
    }
}

// Early fill (decode engine, LRU/ATU): the misses of a step are the list entries whose id has
// no slot yet -- known before the victims are chosen.  k_missq compacts them per tier in
// ascending list order (the order k_lru pairs them with victims), so the host-tier copies can
// start into a staging area while k_lru runs; the miss FFN reads the staging area and the
// records are scattered into their victim slots afterwards (copy stream).
__global__ void __launch_bounds__(NT, 1)
    k_missq(LruArgs a, int32_t *__restrict__ tier_ids, int32_t *__restrict__ q,
            int32_t *__restrict__ qsrc, int32_t *__restrict__ qjob, int F_r, int requant) {
    // q: [16] header (q[8 + t] = misses of tier t) | ids [k] (segments as tier_ids);
    // qsrc (or null): per entry the neuron's FP16-pool slot for an INT8 / INT4 miss whose FP16
    // record is resident (filled by requantisation, k_requant), else -1
    __shared__ int scan_sm[NW];
    extern __shared__ uint32_t bm[];  // [ceil(F_r / 32)]: the tier's ids as a bitmap
    griddep_wait();
    const int tau = blockIdx.x;
    const int n = a.cnt[tau], seg = a.seg[tau];
    const int32_t *slot_of = a.slot_of[tau];
    int32_t *R = tier_ids + seg;
    if (F_r > 0 && n > 1) {
        // the select leaves the tier lists in rank order; ascending ids first (R7: misses are
        // paired with victims in ascending id order): distinct ids in [0, F_r) -> bitmap ->
        // scan of the words' popcounts -> each thread writes its words' ids in order
        const int W = (F_r + 31) >> 5;
        for (int w = threadIdx.x; w < W; w += NT) bm[w] = 0u;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += NT) atomicOr(&bm[R[i] >> 5], 1u << (R[i] & 31));
        __syncthreads();
        const int per = (W + NT - 1) / NT;
        const int w0 = min(W, (int)threadIdx.x * per), w1 = min(W, w0 + per);
        int cnt = 0;
        for (int w = w0; w < w1; w++) cnt += __popc(bm[w]);
        int tot;
        int at = block_scan1(cnt, &tot, scan_sm);
        for (int w = w0; w < w1; w++) {
            uint32_t b = bm[w];
            while (b) {
                const int k = __ffs(b) - 1;
                b &= b - 1;
                R[at++] = (w << 5) + k;
            }
        }
        __syncthreads();  // (the block's global writes are visible to it after the barrier)
    }
    const int CH = (n + NT - 1) / NT;
    const int i0 = min(n, (int)threadIdx.x * CH), i1 = min(n, i0 + CH);
    int nm = 0;
    for (int i = i0; i < i1; i++) nm += slot_of[R[i]] < 0;
    int tot;
    int pos = block_scan1(nm, &tot, scan_sm);
    int nj = 0;  // requantisation jobs of this thread (INT misses resident in the FP16 pool)
    const int pos0 = pos;
    for (int i = i0; i < i1; i++)
        if (slot_of[R[i]] < 0) {
            M2C_CHECK(pos < n && R[i] >= 0 && (F_r == 0 || R[i] < F_r));
            const int s16 = (qsrc && requant && tau > 0) ? a.slot_of[0][R[i]] : -1;
            if (qsrc) qsrc[seg + pos] = s16;
            nj += s16 >= 0;
            q[16 + seg + pos++] = R[i];
        }
    if (qsrc) {  // the jobs' entry indices, compacted in entry order: qjob[seg + j], count q[12 + tau]
        int totj;
        int jpos = block_scan1(nj, &totj, scan_sm);
        for (int m = pos0; m < pos; m++)
            if (qsrc[seg + m] >= 0) qjob[seg + jpos++] = m;
        if (threadIdx.x == 0) q[12 + tau] = totj;
    }
    if (threadIdx.x == 0) q[8 + tau] = tot;
}

struct StageArgs {
    const uint8_t *host[3];   // layer l+1's host tier
    const int32_t *slot_of[3];  // layer l+1's pools (read before layer l+1's lookup)
    int32_t *stage_of[3];     // [F_r] per tier (this parity)
    uint8_t *stage[3];        // [k_t][nb_t] per tier (this parity)
    int32_t *sid;             // [k] staged id per list entry (-1 none)
    int64_t nb[3];
    int seg[3], cnt[3];
};

#ifndef M2C_FILL_U
#define M2C_FILL_U 4  // 16-B loads in flight per lane in k_fill (r02 sweep: 4 x 32 CTAs best)
#endif
struct FillArgs {
    const uint8_t *host[3];
    uint8_t *pool[3];
    int64_t nb[3];
    int seg[3];
    // NEXT-2 lookahead: records staged one layer ahead (device), stage_of[t][id] = index or -1
    const int32_t *stage_of[3];
    const uint8_t *stage[3];
    unsigned long long *staged;  // count of misses filled from the staging buffers
    const int32_t *skip;         // or null: entries with skip[seg + m] >= 0 are not copied
    int32_t *ready;              // or null: ready[seg + m] = fill_tag(*step_ptr, layer) once copied
    const int32_t *step_ptr;
    int layer;
};

// a5: SM-driven gather of the missed records from the pinned host tier (UVA-mapped) into
// their victim slots.  One warp per record, 8 x 16 B loads in flight per lane.
__global__ void __launch_bounds__(256) k_fill(FillArgs a, const int32_t *__restrict__ counts,
                                              const int32_t *__restrict__ miss_ids,
                                              const int32_t *__restrict__ miss_items) {
    griddep_wait();
    const int c0 = counts[8], c1 = counts[9], c2 = counts[10];
    const int total = c0 + c1 + c2;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int w = gw; w < total; w += nwarps) {
        const int tau = w < c0 ? 0 : (w < c0 + c1 ? 1 : 2);
        const int m = w - (tau == 0 ? 0 : (tau == 1 ? c0 : c0 + c1));
        if (a.skip && a.skip[a.seg[tau] + m] >= 0) continue;  // (requantised on the GPU)
        const int id = miss_ids[a.seg[tau] + m];
        const int sl = miss_items[a.seg[tau] + m];
        M2C_CHECK(id >= 0 && sl >= 0);
        const int64_t nv = a.nb[tau] / 16;
        const int si = a.stage_of[tau] ? a.stage_of[tau][id] : -1;  // staged by the lookahead?
        if (si >= 0 && lane == 0) atomicAdd(a.staged, 1ull);
        const uint4 *src = reinterpret_cast<const uint4 *>(
            si >= 0 ? a.stage[tau] + (int64_t)si * a.nb[tau] : a.host[tau] + (int64_t)id * a.nb[tau]);
        uint4 *dst = reinterpret_cast<uint4 *>(a.pool[tau] + (int64_t)sl * a.nb[tau]);
        for (int64_t base = 0; base < nv; base += 32 * M2C_FILL_U) {
            uint4 v[M2C_FILL_U];
#pragma unroll
            for (int j = 0; j < M2C_FILL_U; j++) {
                const int64_t c = base + lane + 32 * j;
                if (c < nv) v[j] = src[c];
            }
#pragma unroll
            for (int j = 0; j < M2C_FILL_U; j++) {
                const int64_t c = base + lane + 32 * j;
                if (c < nv) dst[c] = v[j];
            }
        }
        if (a.ready) {  // the record landed: publish it (release after the warp's stores)
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(a.ready + a.seg[tau] + m),
                             "r"(fill_tag(*a.step_ptr, a.layer))
                             : "memory");
            }
        }
    }
}

// NEXT-2 (the next layer's neurons are predictable from the current layer's input):
// the predicted tier lists of layer l+1 (from x_l) -> the entries that would miss in layer
// l+1's pools now are marked in stage_of (index = position in the tier segment) and copied
// from the host tier into the staging buffers on the copy stream, overlapped with layer l.
// The selection, the cache state and the outputs are unchanged: a miss at layer l+1 whose
// record was staged is filled device-to-device instead of over PCIe.
__global__ void __launch_bounds__(256) k_stage_plan(StageArgs a, const int32_t *__restrict__ spec_ids) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = a.seg[2] + a.cnt[2];
    if (i >= k) return;
    const int tau = i < a.seg[1] ? 0 : (i < a.seg[2] ? 1 : 2);
    const int id = spec_ids[i];
    const bool stage = a.slot_of[tau][id] < 0;
    a.sid[i] = stage ? id : -1;
    if (stage) a.stage_of[tau][id] = i - a.seg[tau];
}

// the staged records: host tier of layer l+1 -> staging buffers (warp per record)
__global__ void __launch_bounds__(256) k_stage_fill(StageArgs a) {
    griddep_wait();
    const int k = a.seg[2] + a.cnt[2];
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int i = gw; i < k; i += nwarps) {
        const int id = a.sid[i];
        if (id < 0) continue;
        const int tau = i < a.seg[1] ? 0 : (i < a.seg[2] ? 1 : 2);
        const int64_t nv = a.nb[tau] / 16;
        const uint4 *src = reinterpret_cast<const uint4 *>(a.host[tau] + (int64_t)id * a.nb[tau]);
        uint4 *dst = reinterpret_cast<uint4 *>(a.stage[tau] + (int64_t)(i - a.seg[tau]) * a.nb[tau]);
        for (int64_t base = 0; base < nv; base += 32 * M2C_FILL_U) {
            uint4 v[M2C_FILL_U];
#pragma unroll
            for (int j = 0; j < M2C_FILL_U; j++) {
                const int64_t c = base + lane + 32 * j;
                if (c < nv) v[j] = src[c];
            }
#pragma unroll
            for (int j = 0; j < M2C_FILL_U; j++) {
                const int64_t c = base + lane + 32 * j;
                if (c < nv) dst[c] = v[j];
            }
        }
    }
}

// after layer l+1's fill consumed them: the staging marks are cleared for reuse
__global__ void __launch_bounds__(256) k_stage_clear(StageArgs a) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = a.seg[2] + a.cnt[2];
    if (i >= k) return;
    const int tau = i < a.seg[1] ? 0 : (i < a.seg[2] ? 1 : 2);
    const int id = a.sid[i];
    if (id >= 0) a.stage_of[tau][id] = -1;
}

}  // namespace

size_t lru_smem_bytes(int P2, int maxcnt) { (void)maxcnt; return 24 * (size_t)P2 + 8 * (size_t)(P2 / 32); }

cudaError_t init_cache_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_lru, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lru_smem_bytes(kMaxPoolSlots, kMaxPoolSlots));
    if (e == cudaSuccess)  // (k_missq's tier-sort bitmap: F_r <= 2^20)
        e = cudaFuncSetAttribute(k_missq, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * (1 << 15));
    return e;
}

cudaError_t launch_lru(m2c_ctx *c, LayerState &L, const int32_t *step_dev, const int32_t *tier_ids,
                       const m2c_tier_plan &p, int32_t *slots, uint32_t *hit_bits,
                       int32_t *miss_log, int32_t *evict_log, cudaStream_t st) {
    LruArgs a;
    const int cnt[3] = {p.k_fp16, p.k_int8, p.k_int4};
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8};
    int P2 = 32, maxcnt = 1;
    for (int t = 0; t < 3; t++) {
        a.occ[t] = L.occupant[t];
        a.last[t] = L.last[t];
        a.slot_of[t] = L.slot_of[t];
        a.ord[t] = L.ord[t];
        a.cap[t] = L.cap[t];
        a.seg[t] = seg[t];
        a.cnt[t] = cnt[t];
        while (P2 < L.cap[t] || P2 < cnt[t]) P2 <<= 1;
        maxcnt = cnt[t] > maxcnt ? cnt[t] : maxcnt;
    }
    // exactly ceil(k/32) words: hit_bits may be the caller's buffer (m2c.h documents that size)
    cudaError_t e = p.k > 0 ? cudaMemsetAsync(hit_bits, 0, sizeof(uint32_t) * ((p.k + 31) / 32), st) : cudaSuccess;
    if (e != cudaSuccess) return e;
    const size_t smem = lru_smem_bytes(P2, maxcnt);
    e = launch_k(k_lru, dim3(3), dim3(NT), smem, st, a, step_dev, tier_ids, slots, hit_bits,
                 c->ws.hit_items, c->ws.miss_items, c->ws.miss_ids, miss_log, evict_log,
                 c->ws.counts, c->ws.stats, P2);
    c->launch_counter++;
    return e;
}

static StageArgs stage_args(m2c_ctx *c, const LayerState &Ln, int par) {
    StageArgs a;
    const m2c_tier_plan &p = c->plan;
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8}, cnt[3] = {p.k_fp16, p.k_int8, p.k_int4};
    for (int t = 0; t < 3; t++) {
        a.host[t] = Ln.host_rec[t];
        a.slot_of[t] = Ln.slot_of[t];
        a.stage_of[t] = c->stage_of[par] + (size_t)t * c->F_r;
        a.stage[t] = c->stage_buf[par][t];
        a.nb[t] = c->nb[t];
        a.seg[t] = seg[t];
        a.cnt[t] = cnt[t];
    }
    a.sid = c->stage_sid[par];
    return a;
}

cudaError_t launch_stage_plan(m2c_ctx *c, const LayerState &Ln, int par, const int32_t *spec_ids,
                              cudaStream_t st) {
    const int k = c->plan.k;
    if (k <= 0) return cudaSuccess;
    cudaError_t e = launch_k(k_stage_plan, dim3((k + 255) / 256), dim3(256), 0, st, stage_args(c, Ln, par), spec_ids);
    c->launch_counter++;
    return e;
}
cudaError_t launch_stage_fill(m2c_ctx *c, const LayerState &Ln, int par, cudaStream_t st) {
    cudaError_t e = launch_k(k_stage_fill, dim3(64), dim3(256), 0, st, stage_args(c, Ln, par));
    c->launch_counter++;
    return e;
}
cudaError_t launch_stage_clear(m2c_ctx *c, const LayerState &Ln, int par, cudaStream_t st) {
    const int k = c->plan.k;
    if (k <= 0) return cudaSuccess;
    cudaError_t e = launch_k(k_stage_clear, dim3((k + 255) / 256), dim3(256), 0, st, stage_args(c, Ln, par));
    c->launch_counter++;
    return e;
}

cudaError_t launch_missq(m2c_ctx *c, const LayerState &L, int32_t *tier_ids,
                         const m2c_tier_plan &p, cudaStream_t st, int32_t *qsrc, bool sort, bool requant) {
    LruArgs a;
    const int cnt[3] = {p.k_fp16, p.k_int8, p.k_int4};
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8};
    for (int t = 0; t < 3; t++) {
        a.slot_of[t] = L.slot_of[t];
        a.seg[t] = seg[t];
        a.cnt[t] = cnt[t];
    }
    const size_t smem = sort ? 4 * (size_t)((c->F_r + 31) / 32) : 0;
    cudaError_t e = launch_k(k_missq, dim3(3), dim3(NT), smem, st, a, tier_ids, c->mq, qsrc,
                             qsrc ? c->mq_job : nullptr, sort ? c->F_r : 0, requant ? 1 : 0);
    c->launch_counter++;
    return e;
}

// generic record copy: dst[t] + dsti[seg + m] * nb  <-  src[t] + srci[seg + m] * nb for the
// counts[8 + t] entries of each tier (k_fill without the lookahead)
cudaError_t launch_copy_recs(m2c_ctx *c, const uint8_t *const src[3], uint8_t *const dst[3],
                             const m2c_tier_plan &p, const int32_t *counts, const int32_t *srci,
                             const int32_t *dsti, cudaStream_t st, const int32_t *skip, int ready_layer) {
    FillArgs a;
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8};
    for (int t = 0; t < 3; t++) {
        a.host[t] = src[t];
        a.pool[t] = dst[t];
        a.nb[t] = c->nb[t];
        a.seg[t] = seg[t];
        a.stage_of[t] = nullptr;
        a.stage[t] = nullptr;
    }
    a.staged = c->ws.stats + 6;
    a.skip = skip;
    a.ready = ready_layer >= 0 ? c->mq_ready : nullptr;
    a.step_ptr = c->ws.counts + 15;
    a.layer = ready_layer;
    static const int fill_ctas = getenv("M2C_FILL_CTAS") ? atoi(getenv("M2C_FILL_CTAS")) : 32;
    cudaError_t e = launch_k(k_fill, dim3(fill_ctas), dim3(256), 0, st, a, counts, srci, dsti);
    c->launch_counter++;
    return e;
}

cudaError_t launch_fill(m2c_ctx *c, const LayerState &L, const m2c_tier_plan &p,
                        cudaStream_t st, int stage_par) {
    FillArgs a;
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8};
    for (int t = 0; t < 3; t++) {
        a.host[t] = L.host_rec[t];
        a.pool[t] = L.pool[t];
        a.nb[t] = c->nb[t];
        a.seg[t] = seg[t];
        a.stage_of[t] = stage_par >= 0 ? c->stage_of[stage_par] + (size_t)t * c->F_r : nullptr;
        a.stage[t] = stage_par >= 0 ? c->stage_buf[stage_par][t] : nullptr;
    }
    a.staged = c->ws.stats + 6;
    a.skip = nullptr;
    a.ready = nullptr;
    a.step_ptr = nullptr;
    a.layer = 0;
    static const int fill_ctas = getenv("M2C_FILL_CTAS") ? atoi(getenv("M2C_FILL_CTAS")) : 32;  // tuning knob
    cudaError_t e = launch_k(k_fill, dim3(fill_ctas), dim3(256), 0, st, a, c->ws.counts, c->ws.miss_ids,
                             c->ws.miss_items);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

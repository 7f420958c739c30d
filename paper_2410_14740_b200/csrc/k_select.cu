// k_select.cu -- a3: top-k by predictor score and the rank -> precision-tier split.
//
// Paper: "Neurons with top-k scores ... are identified as active"; "neurons with
// higher scores are loaded in higher float-point precision"; mix
// 25% FP16 / 25% INT8 / 50% INT4.  Order (score desc, id asc) (R3).
//
// Multi-CTA, single pass, fed by the 4096-bin histogram of (s + smax) >> sh that k_pred_s
// accumulates.  Every CTA (512 threads) redundantly derives the three rank thresholds:
//  1. suffix scan of the histogram -> the bin holding the k16-th, (k16+k8)-th and k-th score;
//  2. one pass over all scores builds 2^sh-bin sub-histograms of those bins -> the exact
//     values V_t and how many of the E_t elements equal to V_t are in (R_t);
//  3. partial ties (R_t < E_t): the tied ids are collected and sorted; the R_t-th smallest
//     is the id cut I_t (ties by ascending id);
// then classifies its own block of 32-id chunks with warp ballots, obtains the tier-list
// positions of its block with a decoupled look-back over the preceding blocks' published
// counts (one 64-bit status word per block, epoch-tagged so it never needs clearing), and
// writes its part of the three ascending id lists (and tier_of).  The last CTA to finish
// clears the histogram for the next layer.  The rank list (API only) is a separate 1-CTA sort.
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int kBins = 4096;
constexpr int kTieCap = 1024;
constexpr int kChunksPerCta = 16;  // 512 ids per CTA

// exclusive block scan of 3 ints per thread (all threads participate)
__device__ __forceinline__ void block_scan3(const int v[3], int ex[3], int tot[3], int *sm /*[3][32]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc[3];
#pragma unroll
    for (int t = 0; t < 3; t++) {
        int x = v[t];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        inc[t] = x;
        if (lane == 31) sm[t * 32 + warp] = x;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int t = 0; t < 3; t++) {
            int x = lane < NW ? sm[t * 32 + lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            sm[t * 32 + lane] = x;
        }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 3; t++) {
        ex[t] = (warp ? sm[t * 32 + warp - 1] : 0) + inc[t] - v[t];
        tot[t] = sm[t * 32 + NW - 1];
    }
    __syncthreads();
}

// bitonic sort of n <= P2 keys in smem (P2 power of two), padded with `pad`; desc or asc
template <typename K>
__device__ __forceinline__ void bitonic(K *a, int n, int P2, K pad, bool desc, int nt) {
    for (int i = n + threadIdx.x; i < P2; i += nt) a[i] = pad;
    __syncthreads();
    for (int size = 2; size <= P2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P2 / 2; i += nt) {
                const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool dir = ((lo & size) == 0) != desc;
                const K x = a[lo], y = a[hi];
                if ((x > y) == dir) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            __syncthreads();
        }
}

// status word: [63:62] state (1 aggregate, 2 inclusive) | [61:56] epoch | 3 x 18-bit counts
__device__ __forceinline__ unsigned long long pack_st(int state, int epoch, int c0, int c1, int c2) {
    return ((unsigned long long)state << 62) | ((unsigned long long)(epoch & 63) << 56) |
           ((unsigned long long)c2 << 36) | ((unsigned long long)c1 << 18) | (unsigned long long)c0;
}

struct SelParams {
    const int32_t *s;
    int *ghist;
    unsigned long long *status;  // [nblk]
    int *done;                   // completion counter (last CTA clears the histogram)
    int *epoch_ptr;              // device launch counter (advanced by the last CTA)
    int F_r, k, k16, k8, smax, sh;
    int32_t *tier_ids;           // [k] three ascending segments
    int8_t *tier_of;             // [F_r] or null
};

__global__ void __launch_bounds__(NT, 1) k_select(SelParams p) {
    extern __shared__ __align__(16) uint8_t smraw[];
    const int nsub = 1 << p.sh;
    int *hist = reinterpret_cast<int *>(smraw);  // [4096]
    int *sub = hist + kBins;                     // [3][nsub]
    int *ties = sub + 3 * nsub;                  // [3][kTieCap]
    __shared__ int scan_sm[96];
    __shared__ int selv[16];
    __shared__ int ntie[3], blk_cnt[NW][3];
    __shared__ int prefix_sh[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int F_r = p.F_r;
    griddep_launch();
    griddep_wait();
    const int epoch = *(volatile const int *)p.epoch_ptr;

    // ---- 1. histogram suffix scan -> bins of the three targets ----
    const int tg[3] = {p.k16, p.k16 + p.k8, p.k};
    constexpr int BPT = kBins / NT;  // 8 bins per thread, descending order
    int lsum = 0;
    {
        int v[BPT];
#pragma unroll
        for (int i = 0; i < BPT; i++) v[i] = p.ghist[kBins - 1 - (tid * BPT + i)];
#pragma unroll
        for (int i = 0; i < BPT; i++) {
            hist[kBins - 1 - (tid * BPT + i)] = v[i];
            lsum += v[i];
        }
    }
    if (tid < 3) ntie[tid] = 0;
    {
        const int vv[3] = {lsum, 0, 0};
        int ex[3], tot[3];
        block_scan3(vv, ex, tot, scan_sm);
        int cum = ex[0];
#pragma unroll
        for (int i = 0; i < BPT; i++) {
            const int b = kBins - 1 - (tid * BPT + i);
            const int v = hist[b];
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (tg[t] > 0 && cum < tg[t] && cum + v >= tg[t]) {
                    selv[t] = b;
                    selv[3 + t] = tg[t] - cum;  // rank needed inside the bin
                }
            cum += v;
        }
    }
    for (int i = tid; i < 3 * nsub; i += NT) sub[i] = 0;
    __syncthreads();
    const int bin0 = tg[0] > 0 ? selv[0] : -1, bin1 = tg[1] > 0 ? selv[1] : -1,
              bin2 = tg[2] > 0 ? selv[2] : -1;
    // ---- 2. sub-histograms of the chosen bins (8 score loads in flight per thread) ----
    for (int n0 = tid; n0 < F_r; n0 += 8 * NT) {
        int v[8];
#pragma unroll
        for (int i = 0; i < 8; i++) v[i] = n0 + i * NT < F_r ? p.s[n0 + i * NT] + p.smax : -1;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (v[i] < 0) continue;
            const int b = v[i] >> p.sh, lo = v[i] & (nsub - 1);
            if (b == bin0) atomicAdd(&sub[lo], 1);
            if (b == bin1) atomicAdd(&sub[nsub + lo], 1);
            if (b == bin2) atomicAdd(&sub[2 * nsub + lo], 1);
        }
    }
    __syncthreads();
    {
        const int SPT = (nsub + NT - 1) / NT;
        int v3[3] = {0, 0, 0}, ex[3], tot[3];
        for (int i = 0; i < SPT; i++) {
            const int c = nsub - 1 - (tid * SPT + i);
            if (c < 0) break;
#pragma unroll
            for (int t = 0; t < 3; t++) v3[t] += sub[t * nsub + c];
        }
        block_scan3(v3, ex, tot, scan_sm);
#pragma unroll
        for (int t = 0; t < 3; t++) {
            if (tg[t] <= 0) continue;
            const int need = selv[3 + t];
            int cum = ex[t];
            for (int i = 0; i < SPT; i++) {
                const int c = nsub - 1 - (tid * SPT + i);
                if (c < 0) break;
                const int v = sub[t * nsub + c];
                if (cum < need && cum + v >= need) {
                    selv[6 + t] = ((t == 0 ? bin0 : (t == 1 ? bin1 : bin2)) << p.sh) | c;  // V_t
                    selv[9 + t] = need - cum;                                            // R_t
                    selv[12 + t] = v;                                                    // E_t
                }
                cum += v;
            }
        }
    }
    __syncthreads();
    int V[3], I[3];
    bool part[3];
#pragma unroll
    for (int t = 0; t < 3; t++) {
        V[t] = tg[t] > 0 ? selv[6 + t] : 0x7fffffff;
        part[t] = tg[t] > 0 && selv[9 + t] < selv[12 + t];
        I[t] = 0x7fffffff;
    }
    // ---- 3. partial ties: the R_t smallest ids among those equal to V_t are in ----
    if (part[0] || part[1] || part[2]) {
        for (int n = tid; n < F_r; n += NT) {
            const int v = p.s[n] + p.smax;
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (part[t] && v == V[t]) {
                    const int q = atomicAdd(&ntie[t], 1);
                    if (q < kTieCap) ties[t * kTieCap + q] = n;
                }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 3; t++) {
            if (!part[t]) continue;
            const int m = ntie[t], R = selv[9 + t];
            if (m <= kTieCap) {
                int P2 = 1;
                while (P2 < m) P2 <<= 1;
                bitonic<int>(ties + t * kTieCap, m, P2, 0x7fffffff, false, NT);
                I[t] = ties[t * kTieCap + R - 1];
                __syncthreads();
            } else {
                // degenerate (e.g. x = 0: every score ties): binary search the smallest id I
                // with #{tied ids <= I} >= R, one block-wide count per step
                int lo = 0, hi = F_r - 1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    int c = 0;
                    for (int nn = tid; nn <= mid; nn += NT) c += (p.s[nn] + p.smax == V[t]);
                    const int vv[3] = {c, 0, 0};
                    int ex[3], tot[3];
                    block_scan3(vv, ex, tot, scan_sm);
                    if (tot[0] >= R) hi = mid;
                    else lo = mid + 1;
                }
                I[t] = lo;
            }
        }
    }
    // ---- 4. classify this CTA's chunks; look back for the tier-list positions ----
    const int Q = (F_r + 31) / 32;
    const int q0 = blockIdx.x * kChunksPerCta;
    int cnt_w[3] = {0, 0, 0};
    int trs = -1;
    unsigned msk[3] = {0, 0, 0};
    const int q = q0 + warp;  // kChunksPerCta == NW: one chunk per warp
    const int n = 32 * q + lane;
    if (q < Q) {
        const int v = n < F_r ? p.s[n] + p.smax : -1;
        bool in[3];
#pragma unroll
        for (int t = 0; t < 3; t++) in[t] = v > V[t] || (v == V[t] && n <= I[t]);
        trs = in[0] ? 0 : (in[1] ? 1 : (in[2] ? 2 : -1));
        if (n >= F_r) trs = -1;
#pragma unroll
        for (int t = 0; t < 3; t++) {
            msk[t] = __ballot_sync(0xffffffffu, trs == t);
            cnt_w[t] = __popc(msk[t]);
        }
    }
    if (lane == 0)
#pragma unroll
        for (int t = 0; t < 3; t++) blk_cnt[warp][t] = cnt_w[t];
    __syncthreads();
    if (warp == 0) {  // exclusive prefix over the CTA's warps (chunks) and block totals
        int c[3];
#pragma unroll
        for (int t = 0; t < 3; t++) {
            int x = lane < NW ? blk_cnt[lane][t] : 0;
            int inc = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane < NW) blk_cnt[lane][t] = inc - x;
            c[t] = __shfl_sync(0xffffffffu, inc, NW - 1);
        }
        if (lane == 0) {  // decoupled look-back
            const int b = blockIdx.x;
            unsigned long long *st = p.status;
            int pre[3] = {0, 0, 0};
            if (b == 0) {
                st[0] = pack_st(2, epoch, c[0], c[1], c[2]);
            } else {
                atomicExch(&st[b], pack_st(1, epoch, c[0], c[1], c[2]));
                for (int j = b - 1; j >= 0; j--) {
                    unsigned long long w;
                    do {
                        w = *((volatile unsigned long long *)&st[j]);
                    } while ((int)((w >> 56) & 63) != (epoch & 63) || (w >> 62) == 0);
                    pre[0] += (int)(w & 0x3ffff);
                    pre[1] += (int)((w >> 18) & 0x3ffff);
                    pre[2] += (int)((w >> 36) & 0x3ffff);
                    if ((w >> 62) == 2) break;
                }
                __threadfence();
                atomicExch(&st[b], pack_st(2, epoch, pre[0] + c[0], pre[1] + c[1], pre[2] + c[2]));
            }
#pragma unroll
            for (int t = 0; t < 3; t++) prefix_sh[t] = pre[t];
        }
    }
    __syncthreads();
    if (q < Q) {
        const int seg[3] = {0, p.k16, p.k16 + p.k8};
        if (n < F_r && p.tier_of) p.tier_of[n] = (int8_t)trs;
        if (trs >= 0) {
            const unsigned lt = (1u << lane) - 1u;
            const unsigned m = trs == 0 ? msk[0] : (trs == 1 ? msk[1] : msk[2]);
            const int pos = prefix_sh[trs] + blk_cnt[warp][trs] + __popc(m & lt);
            M2C_CHECK(pos >= 0 && pos < (trs == 0 ? p.k16 : (trs == 1 ? p.k8 : p.k - p.k16 - p.k8)));
            p.tier_ids[seg[trs] + pos] = n;
        }
    }
    // ---- the last CTA clears the histogram for the next layer ----
    __syncthreads();
    __shared__ int last;
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(p.done, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last) {  // every CTA has read the histogram and the epoch: reset for the next launch
        for (int i = tid; i < kBins; i += NT) p.ghist[i] = 0;
        if (tid == 0) {
            *p.done = 0;
            *p.epoch_ptr = (epoch + 1) & 63;
        }
    }
}

// API path: the rank list = the selected ids sorted by (score desc, id asc)
__global__ void __launch_bounds__(1024, 1)
    k_rank_list(const int32_t *__restrict__ s, const int32_t *__restrict__ tier_ids, int k,
                int P2, int32_t *__restrict__ rank_list) {
    extern __shared__ __align__(16) unsigned long long ck[];
    griddep_wait();
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const int n = tier_ids[i];
        ck[i] = ((unsigned long long)((uint32_t)s[n] ^ 0x80000000u) << 32) | (uint32_t)(~(uint32_t)n);
    }
    __syncthreads();
    bitonic<unsigned long long>(ck, k, P2, 0ull, true, blockDim.x);
    for (int i = threadIdx.x; i < k; i += blockDim.x) rank_list[i] = (int32_t)(~(uint32_t)(ck[i] & 0xffffffffu));
}

}  // namespace

size_t select_smem_bytes(int sh) { return 4 * ((size_t)kBins + 3 * ((size_t)1 << sh) + 3 * (size_t)kTieCap); }
int select_blocks(int F_r) { return ((F_r + 31) / 32 + kChunksPerCta - 1) / kChunksPerCta; }

// ---- NEXT-3: exact global top-k under d_ff sharding (P:253 global top-k semantics) --------
// Each rank sends its local top-n candidates as 64-bit keys (score << 32 | ~global id): the
// descending key order is (score desc, global id asc), R3.  Because a rank can contribute at
// most k of the global top-k, n = min(F_r, k_global) candidates per rank make the union exact.
__global__ void __launch_bounds__(256) k_cand_keys(const int32_t *__restrict__ s,
                                                   const int32_t *__restrict__ rank_list, int n, int gbase,
                                                   long long *__restrict__ keys) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int id = rank_list[i];
    keys[i] = (long long)(((unsigned long long)(unsigned)s[id] << 32) | (unsigned)~(unsigned)(gbase + id));
}

// One CTA: the P gathered runs (each sorted descending) -> the three global cuts by bisection on
// the key value (warp t, lane r binary-searches run r; counts by warp sums), then this rank's
// run segments [K_t, K_{t-1}) -> local ids ascending per tier (rank by id inside a segment).
__global__ void __launch_bounds__(1024) k_select_global(const long long *__restrict__ keys, int P, int n,
                                                        int rank, int F_r, int k16, int k8, int k,
                                                        int32_t *__restrict__ tier_ids,
                                                        int32_t *__restrict__ counts) {
    extern __shared__ __align__(16) long long runs[];  // [P][n]
    __shared__ long long cut[3];
    __shared__ int seg[4];
    griddep_wait();
    for (int i = threadIdx.x; i < P * n; i += blockDim.x) runs[i] = keys[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto count_ge = [&](int r, long long X) {  // keys >= X in run r
        int a = 0, b = n;
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (runs[r * n + mid] >= X) a = mid + 1;
            else b = mid;
        }
        return a;
    };
    if (warp < 3) {
        const int t = warp;
        const int target = t == 0 ? k16 : (t == 1 ? k16 + k8 : k);
        long long K = 0x7fffffffffffffffll;  // empty cut: no key reaches it
        if (target > 0) {
            // the target-th largest key: largest X with #(keys >= X) >= target (keys distinct)
            long long lo = -(1ll << 60), hi = 1ll << 60;  // |key| < 2^56 (|s| < 2^24)
            while (lo < hi) {
                const long long mid = lo + (long long)(((unsigned long long)(hi - lo) + 1ull) >> 1);
                int c = lane < P ? count_ge(lane, mid) : 0;
                c = __reduce_add_sync(0xffffffffu, c);
                if (c >= target) lo = mid;
                else hi = mid - 1;
            }
            K = lo;
        }
        if (lane == 0) cut[t] = K;
    }
    __syncthreads();
    if (threadIdx.x < 3) seg[threadIdx.x + 1] = count_ge(rank, cut[threadIdx.x]);  // nested prefixes
    if (threadIdx.x == 0) seg[0] = 0;
    __syncthreads();
    const int base = rank * F_r;
    const int off[3] = {0, k16, k16 + k8};
    for (int t = 0; t < 3; t++) {
        const int a = seg[t], b = seg[t + 1];
        for (int e = a + (int)threadIdx.x; e < b; e += blockDim.x) {
            const unsigned gid = ~(unsigned)(runs[rank * n + e] & 0xffffffffll);
            int rk = 0;  // members with a smaller id come first
            for (int e2 = a; e2 < b; e2++) rk += ~(unsigned)(runs[rank * n + e2] & 0xffffffffll) < gid;
            tier_ids[off[t] + rk] = (int)gid - base;
        }
        if (threadIdx.x == 0) counts[t] = b - a;
    }
}

cudaError_t init_select_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)select_smem_bytes(12));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_rank_list, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    return e;
}

cudaError_t launch_cand_keys(m2c_ctx *c, const int32_t *scores, const int32_t *rank_list, int n,
                             long long *keys, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    cudaError_t e = launch_k(k_cand_keys, dim3((n + 255) / 256), dim3(256), 0, st, scores, rank_list, n,
                             c->desc.shard_index * c->F_r, keys);
    c->launch_counter++;
    return e;
}

cudaError_t launch_select_global(m2c_ctx *c, const long long *keys, int n, const m2c_tier_plan &g,
                                 int32_t *tier_ids, int32_t *counts, cudaStream_t st) {
    const size_t smem = 8 * (size_t)c->desc.shard_count * n;
    cudaError_t e = cudaFuncSetAttribute(k_select_global, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_k(k_select_global, dim3(1), dim3(1024), smem, st, keys, c->desc.shard_count, n,
                 c->desc.shard_index, c->F_r, g.k_fp16, g.k_int8, g.k, tier_ids, counts);
    c->launch_counter++;
    return e;
}

cudaError_t launch_select(m2c_ctx *c, const int32_t *scores, int *hist, const m2c_tier_plan &p,
                          int32_t *rank_list, int8_t *tier_of, int32_t *tier_ids, cudaStream_t st) {
    cudaError_t e;
    SelParams sp;
    sp.s = scores;
    sp.ghist = hist;
    sp.status = c->sel_status;
    sp.done = c->sel_done;
    sp.epoch_ptr = c->sel_epoch;
    sp.F_r = c->F_r;
    sp.k = p.k;
    sp.k16 = p.k_fp16;
    sp.k8 = p.k_int8;
    sp.smax = c->sel_smax;
    sp.sh = c->sel_sh;
    sp.tier_ids = tier_ids;
    sp.tier_of = tier_of;
    e = launch_k(k_select, dim3(select_blocks(c->F_r)), dim3(NT), select_smem_bytes(c->sel_sh), st, sp);
    c->launch_counter++;
    if (e != cudaSuccess || rank_list == nullptr || p.k == 0) return e;
    int P2 = 2;
    while (P2 < p.k) P2 <<= 1;
    e = launch_k(k_rank_list, dim3(1), dim3(1024), 8 * (size_t)P2, st, scores, tier_ids, p.k, P2, rank_list);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

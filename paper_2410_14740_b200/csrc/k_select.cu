// k_select.cu -- a3: top-k by predictor score and the rank -> precision-tier split.
//
// Paper: "Neurons with top-k scores ... are identified as active"; "neurons with
// higher scores are loaded in higher float-point precision"; mix
// 25% FP16 / 25% INT8 / 50% INT4.  Order (score desc, id asc) (R3).
//
// One CTA of 1024 threads.  Scores -> order-preserving uint32 keys in smem.  The three rank
// thresholds (k16-th, (k16+k8)-th, k-th largest key) are found by an MSB-first radix select
// that starts at the highest bit where min and max key differ (the predictor scores span
// ~20 of the 32 bits), uses one shared 256-bin histogram for the first digit (the three
// searches share an empty prefix) and afterwards iterates only over a compacted candidate
// list (the elements inside the chosen bins).  Ties at a threshold are resolved by ascending
// id with a block scan; a second scan compacts the three tiers into ascending id lists.
// Optional rank_list: bitonic sort of the k selected (key, ~id) composites.
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int NT = kSelectThreads;
constexpr int NW = NT / 32;
constexpr int kMaxCand = 2048;  // candidate list capacity (falls back to a full scan beyond)

// exclusive block scan of 3 ints per thread (all threads participate)
__device__ __forceinline__ void block_scan3(int v[3], int excl[3], int tot[3], int *sm /*[3][NW]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc[3];
#pragma unroll
    for (int t = 0; t < 3; t++) {
        int x = v[t];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        inc[t] = x;
        if (lane == 31) sm[t * NW + warp] = x;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int t = 0; t < 3; t++) {
            int x = (lane < NW) ? sm[t * NW + lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane < NW) sm[t * NW + lane] = x;  // inclusive warp totals
        }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 3; t++) {
        const int wbase = warp ? sm[t * NW + warp - 1] : 0;
        excl[t] = wbase + inc[t] - v[t];
        tot[t] = sm[t * NW + NW - 1];
    }
    __syncthreads();
}

// warp w < 3 finds, in hist[w] (scanned from the top bin), the bin holding the need-th
// element; writes the new prefix bits and the remaining rank.
__device__ __forceinline__ void pick_bin(const int *hist, int need, uint32_t prefix, int shift,
                                         uint32_t *out_prefix, int *out_rem) {
    const int lane = threadIdx.x & 31;
    int loc[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        loc[j] = hist[255 - 8 * lane - j];
        sum += loc[j];
    }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const int excl = inc - sum;
    const unsigned ball = __ballot_sync(0xffffffffu, inc >= need);
    const int src = __ffs(ball) - 1;
    if (lane == src) {
        int cum = excl, b = -1, before = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (b < 0 && cum + loc[j] >= need) {
                b = 255 - 8 * lane - j;
                before = cum;
            }
            cum += loc[j];
        }
        *out_prefix = prefix | ((uint32_t)b << shift);
        *out_rem = need - before;
    }
}

__global__ void __launch_bounds__(NT, 1)
    k_select(int F_r, const int32_t *__restrict__ s, int k, int k16, int k8,
             int32_t *__restrict__ rank_list, int8_t *__restrict__ tier_of,
             int32_t *__restrict__ tier_ids, int P2) {
    extern __shared__ __align__(16) uint8_t smraw[];
    uint32_t *keys = reinterpret_cast<uint32_t *>(smraw);                     // [F_r]
    int8_t *tier = reinterpret_cast<int8_t *>(smraw + 4 * ((F_r + 3) & ~3));  // [F_r]
    unsigned long long *ck = reinterpret_cast<unsigned long long *>(
        smraw + 4 * ((F_r + 3) & ~3) + ((F_r + 15) & ~15));                      // [P2]
    __shared__ int hist[3][256];
    __shared__ int scan_sm[3 * NW];
    __shared__ uint32_t sel_prefix[3], mm[2 * NW];
    __shared__ int sel_rem[3];
    __shared__ uint32_t cand[3][kMaxCand];
    __shared__ int ncand[3];
    griddep_wait();

    uint32_t kmin = 0xffffffffu, kmax = 0;
    for (int n = threadIdx.x; n < F_r; n += NT) {
        const uint32_t key = (uint32_t)s[n] ^ 0x80000000u;
        keys[n] = key;
        kmin = min(kmin, key);
        kmax = max(kmax, key);
    }
    for (int i = threadIdx.x; i < 3 * 256; i += NT) (&hist[0][0])[i] = 0;
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        mm[warp] = kmin;
        mm[NW + warp] = kmax;
    }
    if (threadIdx.x < 3) ncand[threadIdx.x] = 0;
    __syncthreads();
    if (warp == 0) {  // one warp folds the per-warp extrema, then broadcasts through smem
        const uint32_t a = __reduce_min_sync(0xffffffffu, lane < NW ? mm[lane] : 0xffffffffu);
        const uint32_t b = __reduce_max_sync(0xffffffffu, lane < NW ? mm[NW + lane] : 0u);
        if (lane == 0) {
            mm[0] = a;
            mm[1] = b;
        }
    }
    __syncthreads();
    kmin = mm[0];
    kmax = mm[1];
    const int target[3] = {k16, k16 + k8, k};
    const uint32_t diff = kmin ^ kmax;
    // highest varying bit hb; digit passes cover bits [0, hb]; bits above are common
    const int hb = diff ? 31 - __clz(diff) : 0;
    int shift = hb >= 7 ? hb - 7 : 0;
    uint32_t mask = diff ? ~((2u << hb) - 1u) : 0xffffffffu;  // hb == 31 -> mask 0
    if (hb == 31) mask = 0;
    const uint32_t common = kmin & mask;
    uint32_t prefix[3] = {common, common, common};
    int rem[3] = {target[0], target[1], target[2]};

    // ---- pass 1: one histogram over all keys (shared by the three searches) ----
    if (k > 0 && diff) {
        for (int n = threadIdx.x; n < F_r; n += NT) atomicAdd(&hist[0][(keys[n] >> shift) & 255], 1);
        __syncthreads();
        if (warp < 3 && rem[warp] > 0)
            pick_bin(hist[0], rem[warp], prefix[warp], shift, &sel_prefix[warp], &sel_rem[warp]);
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 3; t++)
            if (rem[t] > 0) {
                prefix[t] = sel_prefix[t];
                rem[t] = sel_rem[t];
            }
        mask |= 255u << shift;
        // ---- compact the candidates of each search (keys inside the chosen bin) ----
        for (int n = threadIdx.x; n < F_r; n += NT) {
            const uint32_t key = keys[n];
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (rem[t] > 0 && (key & mask) == prefix[t]) {
                    const int p = atomicAdd(&ncand[t], 1);
                    if (p < kMaxCand) cand[t][p] = key;
                }
        }
        __syncthreads();
        // ---- remaining digits over the candidate lists only ----
        while (shift > 0) {
            const int nshift = shift >= 8 ? shift - 8 : 0;
            const uint32_t dmask = ((1u << (shift - nshift)) - 1u);
            for (int i = threadIdx.x; i < 3 * 256; i += NT) (&hist[0][0])[i] = 0;
            __syncthreads();
#pragma unroll
            for (int t = 0; t < 3; t++) {
                if (rem[t] <= 0) continue;
                const int nc = ncand[t];
                if (nc <= kMaxCand) {
                    for (int i = threadIdx.x; i < nc; i += NT) {
                        const uint32_t key = cand[t][i];
                        if ((key & mask) == prefix[t]) atomicAdd(&hist[t][(key >> nshift) & dmask], 1);
                    }
                } else {  // overflowed candidate list: scan every key
                    for (int n = threadIdx.x; n < F_r; n += NT) {
                        const uint32_t key = keys[n];
                        if ((key & mask) == prefix[t]) atomicAdd(&hist[t][(key >> nshift) & dmask], 1);
                    }
                }
            }
            __syncthreads();
            if (warp < 3 && rem[warp] > 0)
                pick_bin(hist[warp], rem[warp], prefix[warp], nshift, &sel_prefix[warp], &sel_rem[warp]);
            __syncthreads();
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (rem[t] > 0) {
                    prefix[t] = sel_prefix[t];
                    rem[t] = sel_rem[t];
                }
            mask |= dmask << nshift;
            shift = nshift;
        }
    } else if (k > 0) {  // all keys equal: the threshold is that key, ties by id
#pragma unroll
        for (int t = 0; t < 3; t++) prefix[t] = kmin;
    }
    // now: element n has rank < target[t] iff key > prefix[t], or key == prefix[t] and it is
    // among the first rem[t] such elements in ascending id order (target 0: nobody).

    // ---- classify (needs the running count of equal keys in id order) ----
    const int CH = (F_r + NT - 1) / NT;
    const int n0 = min(F_r, (int)threadIdx.x * CH), n1 = min(F_r, n0 + CH);
    int v[3], ex[3], tot[3];
#pragma unroll
    for (int t = 0; t < 3; t++) v[t] = 0;
    for (int n = n0; n < n1; n++) {
        const uint32_t key = keys[n];
#pragma unroll
        for (int t = 0; t < 3; t++) v[t] += (target[t] > 0 && key == prefix[t]);
    }
    block_scan3(v, ex, tot, scan_sm);
    int cnt[3] = {0, 0, 0};
    for (int n = n0; n < n1; n++) {
        const uint32_t key = keys[n];
        int tr = -1;
#pragma unroll
        for (int t = 2; t >= 0; t--) {
            bool in = false;
            if (target[t] > 0) {
                if (key > prefix[t]) in = true;
                else if (key == prefix[t]) in = (ex[t]++ < rem[t]);
            }
            if (in) tr = t;
        }
        tier[n] = (int8_t)tr;
        if (tr >= 0) cnt[tr]++;
    }
    // ---- compact the tiers into ascending id lists ----
    block_scan3(cnt, ex, tot, scan_sm);
    const int seg[3] = {0, k16, k16 + k8};
    for (int n = n0; n < n1; n++) {
        const int tr = tier[n];
        if (tier_of) tier_of[n] = (int8_t)tr;
        if (tr >= 0) tier_ids[seg[tr] + ex[tr]++] = n;
    }
    griddep_launch();
    if (rank_list == nullptr || k == 0) return;

    // ---- rank list: bitonic sort (descending) of the selected (key, ~id) composites ----
    __syncthreads();
    int c3[3] = {0, 0, 0};
    for (int n = n0; n < n1; n++) c3[0] += (tier[n] >= 0);
    block_scan3(c3, ex, tot, scan_sm);
    int pos = ex[0];
    for (int n = n0; n < n1; n++)
        if (tier[n] >= 0)
            ck[pos++] = ((unsigned long long)keys[n] << 32) | (uint32_t)(~(uint32_t)n);
    for (int i = k + (int)threadIdx.x; i < P2; i += NT) ck[i] = 0ull;
    __syncthreads();
    for (int size = 2; size <= P2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P2 / 2; i += NT) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool desc = ((lo & size) == 0);
                const unsigned long long a = ck[lo], b = ck[hi];
                if ((a < b) == desc) {
                    ck[lo] = b;
                    ck[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < k; i += NT) rank_list[i] = (int32_t)(~(uint32_t)(ck[i] & 0xffffffffu));
}

}  // namespace

size_t select_smem_bytes(int F_r, int P2) {
    return 4 * (size_t)((F_r + 3) & ~3) + (size_t)((F_r + 15) & ~15) + 8 * (size_t)P2;
}

static size_t g_select_smem_max = 0;

cudaError_t init_select_attrs() {
    // opt-in limit per block minus this kernel's static shared memory
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k_select);
    if (e != cudaSuccess) return e;
    g_select_smem_max = (size_t)optin - fa.sharedSizeBytes;
    return cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)g_select_smem_max);
}

size_t select_smem_limit() { return g_select_smem_max; }

cudaError_t launch_select(m2c_ctx *c, const int32_t *scores, const m2c_tier_plan &p,
                          int32_t *rank_list, int8_t *tier_of, int32_t *tier_ids,
                          cudaStream_t st) {
    int P2 = 0;
    if (rank_list && p.k > 0) {
        P2 = 1;
        while (P2 < p.k) P2 <<= 1;
        if (P2 < 2) P2 = 2;
    }
    const size_t smem = select_smem_bytes(c->F_r, P2);
    cudaError_t e = launch_k(k_select, dim3(1), dim3(NT), smem, st, c->F_r, scores, p.k, p.k_fp16,
                             p.k_int8, rank_list, tier_of, tier_ids, P2);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

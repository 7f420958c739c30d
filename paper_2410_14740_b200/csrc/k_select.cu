// k_select.cu -- a3: top-k by predictor score and the rank -> precision-tier split.
//
// Paper: "Neurons with top-k scores ... are identified as active"; "neurons with
// higher scores are loaded in higher float-point precision"; mix
// 25% FP16 / 25% INT8 / 50% INT4.  Order (score desc, id asc) (R3).
//
// One CTA: scores -> order-preserving uint32 keys in smem; three simultaneous MSB-first radix
// selects (8-bit digits) find the k16-th, (k16+k8)-th and k-th largest key and how many of
// the elements equal to it are inside (ties are resolved by ascending id through a block
// scan); then a second block scan compacts the three tiers into ascending id lists.
// Optional rank_list: bitonic sort of the k selected (key, ~id) composites.
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int NT = kSelectThreads;
constexpr int NW = NT / 32;

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
    __shared__ uint32_t sel_prefix[3];
    __shared__ int sel_rem[3];
    griddep_wait();

    for (int n = threadIdx.x; n < F_r; n += NT) keys[n] = (uint32_t)s[n] ^ 0x80000000u;
    const int target[3] = {k16, k16 + k8, k};
    uint32_t prefix[3] = {0, 0, 0}, mask = 0;
    int rem[3] = {target[0], target[1], target[2]};
    __syncthreads();

    // ---- three simultaneous radix selects (MSB first, 8-bit digits) ----
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 3 * 256; i += NT) (&hist[0][0])[i] = 0;
        __syncthreads();
        for (int n = threadIdx.x; n < F_r; n += NT) {
            const uint32_t key = keys[n];
            const int dg = (key >> shift) & 255;
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (rem[t] > 0 && (key & mask) == prefix[t]) atomicAdd(&hist[t][dg], 1);
        }
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp < 3 && rem[warp] > 0) {
            // lane covers bins [255-8*lane-7, 255-8*lane], scanned from the top
            int loc[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                loc[j] = hist[warp][255 - 8 * lane - j];
                sum += loc[j];
            }
            int inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const int excl = inc - sum;
            const int need = rem[warp];
            const unsigned ball = __ballot_sync(0xffffffffu, inc >= need);
            const int src = __ffs(ball) - 1;  // first lane whose cumulative count reaches need
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
                sel_prefix[warp] = prefix[warp] | ((uint32_t)b << shift);
                sel_rem[warp] = need - before;
            }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 3; t++)
            if (rem[t] > 0) {
                prefix[t] = sel_prefix[t];
                rem[t] = sel_rem[t];
            }
        mask |= 255u << shift;
        __syncthreads();
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
    if (rank_list == nullptr || k == 0) return;

    // ---- rank list: bitonic sort (descending) of the selected (key, ~id) composites ----
    __syncthreads();
    // positions of the selected in id order: reuse the tier counts scan
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
    cudaError_t e = launch_k(k_select, dim3(1), dim3(NT), smem, st, c->F_r, scores, p.k, p.k_fp16, p.k_int8,
                 rank_list, tier_of, tier_ids, P2);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

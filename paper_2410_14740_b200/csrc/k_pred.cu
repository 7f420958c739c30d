// k_pred.cu -- a1/a2: the low-rank neuron-score predictor.
//
// Paper: "A low-rank predictor locates the necessary neurons" (P:73 step 1), one predictor per
// layer driven by the layer's input, assigning "a predicted score to each neuron"
// (Deja Vu).  Form and precision are unspecified; R2: s = B * Q(A x) with
// INT8 factors and exact integer arithmetic: x_j 2^24 is an integer for every fp16 x_j, so
// h = A x is an exact int64 (|h| < 2^60), hq = Q(h) is exact, and s = B hq (dp4a, int32).
// Scores are therefore bit-identical for any reduction order -- h is formed by integer
// atomics from column slices (each CTA owns 32 columns of A, i.e. 32 rows of A^T), which is
// exactly how the persistent decode kernel forms it inside the previous layer's reduction.
//
// Q(v)_i = sgn(v_i) floor((254 |v_i| + M) / (2M)), M = max |v| (quant127_u64: fp64 estimate,
// two 128-bit integer checks).
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kHCols = 32;  // columns of A (rows of A^T) per CTA
constexpr int kHThreads = 256;
constexpr int kSThreads = 256;

// a1: h += A[:, 32 c .. 32 c + 32) x[32 c .. 32 c + 32) for CTA c (h zeroed by the caller).
__global__ void __launch_bounds__(kHThreads) k_pred_h(int d, int r, const __half *__restrict__ x,
                                                      const int8_t *__restrict__ At,
                                                      long long *__restrict__ h, uint32_t *err,
                                                      PrefetchArgs pf) {
    __shared__ int xm[kHCols], xsh[kHCols];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * kHCols;
    // independent of the predecessor: pull this CTA's rows of A^T towards L2, and (decode path)
    // this CTA's share of the records the previous token selected for this layer -- ~80% of
    // them recur and will be read by this layer's FFN; then let the next kernel
    // launch and wait for x
    if (threadIdx.x == 0) prefetch_l2(At + (int64_t)j0 * r, (uint32_t)(kHCols * r));
    if (pf.prev_ids && warp == kHThreads / 32 - 1) {
        const int k = pf.k[0] + pf.k[1] + pf.k[2];
        const int i0 = (int)((long long)k * blockIdx.x / gridDim.x);
        const int i1 = (int)((long long)k * (blockIdx.x + 1) / gridDim.x);
        for (int i = i0 + lane; i < i1; i += 32) {
            const int t = i < pf.k[0] ? 0 : (i < pf.k[0] + pf.k[1] ? 1 : 2);
            const int id = pf.prev_ids[i];
            if (id >= 0 && id < pf.F_r) prefetch_l2(pf.pool[t] + (int64_t)id * pf.nb[t], (uint32_t)pf.nb[t]);
        }
    }
    griddep_launch();
    griddep_wait();
    if (threadIdx.x < kHCols) {
        const unsigned b = __half_as_ushort(x[j0 + threadIdx.x]);
        bool bad = false;
        int m, sh;
        fp16_fixed(b, m, sh, bad);
        if (bad) flag_error(err, 1u);  // Inf / NaN input: flagged, contributes 0
        xm[threadIdx.x] = m;
        xsh[threadIdx.x] = sh;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < r; i += kHThreads) {
        const int8_t *col = At + (int64_t)j0 * r + i;
        int av[kHCols];
#pragma unroll
        for (int j = 0; j < kHCols; j++) av[j] = __ldg(col + (int64_t)j * r);
        unsigned long long acc = 0;
#pragma unroll
        for (int j = 0; j < kHCols; j++) acc += (unsigned long long)(long long)(av[j] * xm[j]) << xsh[j];
        if (acc) red_add_u64(h + (int64_t)i * kHStride, (long long)acc);
    }
}

// a2: hq = Q(h) (every CTA, redundantly), s = B hq for this CTA's rows; LPR lanes per row.
// Decode path: also the 4096-bin histogram of (s + smax) >> sh for the select kernel.
template <int LPR>
__global__ void __launch_bounds__(kSThreads) k_pred_s(int r, int F_r, int rows_per_cta,
                                                      const long long *__restrict__ h,
                                                      const int8_t *__restrict__ B,
                                                      int32_t *__restrict__ s, int *__restrict__ hist,
                                                      int smax, int sh) {
    __shared__ __align__(16) int8_t hq[512];
    __shared__ unsigned long long red[kSThreads / 32];
    const int base = blockIdx.x * rows_per_cta;
    const int rows = min(rows_per_cta, F_r - base);
    if (threadIdx.x == 0 && rows > 0) prefetch_l2(B + (int64_t)base * r, (uint32_t)(rows * r));
    griddep_launch();
    griddep_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int RPW = 32 / LPR;                     // rows per warp per pass
    constexpr int RPP = RPW * (kSThreads / 32);       // rows per pass
    const int part = lane % LPR, sub = lane / LPR;
    // issue this thread's B loads first (independent of h)
    constexpr int kMaxPass = 8;
    int4 bv[kMaxPass];
#pragma unroll
    for (int i = 0; i < kMaxPass; i++) {
        const int rl = i * RPP + warp * RPW + sub;
        bv[i] = (rl < rows) ? __ldg(reinterpret_cast<const int4 *>(B + (int64_t)(base + rl) * r) + part)
                            : make_int4(0, 0, 0, 0);
    }
    unsigned long long mh = 0;
    for (int i = threadIdx.x; i < r; i += kSThreads) {
        const long long v = __ldcg(h + (int64_t)i * kHStride);
        mh = max(mh, (unsigned long long)(v < 0 ? -v : v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, o));
    if (lane == 0) red[warp] = mh;
    __syncthreads();
    mh = red[0];
#pragma unroll
    for (int w = 1; w < kSThreads / 32; w++) mh = max(mh, red[w]);
    for (int i = threadIdx.x; i < r; i += kSThreads) {
        const long long v = __ldcg(h + (int64_t)i * kHStride);
        const int q = quant127_u64((unsigned long long)(v < 0 ? -v : v), mh);
        hq[i] = (int8_t)(v < 0 ? -q : q);
    }
    __syncthreads();
    const int4 hv4 = reinterpret_cast<const int4 *>(hq)[part];
#pragma unroll
    for (int i = 0; i < kMaxPass; i++) {
        const int rl = i * RPP + warp * RPW + sub;
        int acc = 0;
        acc = __dp4a(bv[i].x, hv4.x, acc);
        acc = __dp4a(bv[i].y, hv4.y, acc);
        acc = __dp4a(bv[i].z, hv4.z, acc);
        acc = __dp4a(bv[i].w, hv4.w, acc);
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (part == 0 && rl < rows) {
            s[base + rl] = acc;
            if (hist) atomicAdd(&hist[(acc + smax) >> sh], 1);
        }
    }
}

}  // namespace

cudaError_t launch_predict(m2c_ctx *c, const LayerState &L, const __half *x, int32_t *scores,
                           int *hist, const int32_t *prefetch_ids, cudaStream_t st) {
    const int d = c->desc.d_model, r = c->desc.pred_rank, F_r = c->F_r;
    PrefetchArgs pf;
    pf.prev_ids = prefetch_ids;
    pf.F_r = F_r;
    pf.k[0] = c->plan.k_fp16;
    pf.k[1] = c->plan.k_int8;
    pf.k[2] = c->plan.k_int4;
    for (int t = 0; t < 3; t++) {
        pf.pool[t] = L.pool[t];
        pf.nb[t] = (int)c->nb[t];
    }
    cudaError_t e = cudaMemsetAsync(c->ws.h, 0, sizeof(long long) * kHStride * (size_t)r, st);
    if (e != cudaSuccess) return e;
    e = launch_k(k_pred_h, dim3(d / kHCols), dim3(kHThreads), 0, st, d, r, x, L.A, c->ws.h, c->ws.err, pf);
    if (e != cudaSuccess) return e;
    c->launch_counter++;
    // rows per CTA: at most one pass set (8 passes) per thread, at most one CTA per SM
    const int lpr = r / 16, rpp = (32 / lpr) * (kSThreads / 32);
    int rows = (F_r + c->num_sms - 1) / c->num_sms;
    rows = (rows + rpp - 1) / rpp * rpp;
    if (rows > 8 * rpp) rows = 8 * rpp;
    const dim3 grid((F_r + rows - 1) / rows), block(kSThreads);
    const int sm = c->sel_smax, sh = c->sel_sh;
    switch (lpr) {
        case 1: e = launch_k(k_pred_s<1>, grid, block, 0, st, r, F_r, rows, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 2: e = launch_k(k_pred_s<2>, grid, block, 0, st, r, F_r, rows, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 4: e = launch_k(k_pred_s<4>, grid, block, 0, st, r, F_r, rows, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 8: e = launch_k(k_pred_s<8>, grid, block, 0, st, r, F_r, rows, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 16: e = launch_k(k_pred_s<16>, grid, block, 0, st, r, F_r, rows, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 32: e = launch_k(k_pred_s<32>, grid, block, 0, st, r, F_r, rows, c->ws.h, L.B, scores, hist, sm, sh); break;
        default: return cudaErrorInvalidValue;
    }
    c->launch_counter++;
    return e;
}

}  // namespace m2c

// k_pred.cu -- a1/a2: the low-rank neuron-score predictor.
//
// Paper: "A low-rank predictor locates the necessary neurons" (P:73 step 1), one predictor per
// layer driven by the layer's input, assigning "a predicted score to each neuron"
// (Deja Vu).  Form and precision are unspecified; R2: s = B * Q(A * Q(x))
// with INT8 factors and exact integer arithmetic (dp4a, int32 accumulation), so scores are
// bit-identical for any reduction order.
//
// Q(v)_j = sgn(v_j) floor((254 |v_j| + M) / (2M)), M = max |v|, is computed exactly without
// integer division: q0 = floor(127 |v| / M + 1/2) in fp32 is within one of the answer, and the
// sign of 254 |v| - (2 q0 -+ 1) M, evaluated by one FMA (exact product, single rounding that
// cannot flip a sign), decides the +-1 correction.  For x the operands are fp16 values, so
// 254 |x| and M are exact in fp32; for h (int32) the same test runs in fp64.
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kHRowsPerCta = 2;  // rows of A per CTA (4 warps per row)
constexpr int kHThreads = 256;
constexpr int kSThreads = 256;

__device__ __forceinline__ int q127_f32(float a, float M, float inv) {  // a = |v| >= 0, M > 0
    int q = (int)fmaf(a, inv, 0.5f);
    const float a254 = 254.f * a;  // exact: a is an fp16 value
    if (fmaf(-(float)(2 * q - 1), M, a254) < 0.f) q -= 1;
    else if (fmaf(-(float)(2 * q + 1), M, a254) >= 0.f) q += 1;
    return q;
}
__device__ __forceinline__ int q127_f64(double a, double M, double inv) {
    int q = (int)fma(a, inv, 0.5);
    const double a254 = 254.0 * a;
    if (fma(-(double)(2 * q - 1), M, a254) < 0.0) q -= 1;
    else if (fma(-(double)(2 * q + 1), M, a254) >= 0.0) q += 1;
    return q;
}

// a1: xq = Q(x) (every CTA, redundantly: d <= 8K halves from L2), h = A xq for 2 rows.
__global__ void __launch_bounds__(kHThreads) k_pred_h(int d, int r, const __half *__restrict__ x,
                                                      const int8_t *__restrict__ A,
                                                      int32_t *__restrict__ h, uint32_t *err,
                                                      PrefetchArgs pf) {
    extern __shared__ __align__(16) int8_t xq[];
    __shared__ unsigned red_u[kHThreads / 32];
    __shared__ int red_i[kHThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // independent of the predecessor: pull this CTA's rows of A towards L2, and (decode path)
    // this CTA's share of the records the previous token selected for this layer -- ~80% of
    // them recur and will be read by this layer's FFN; then let the next kernel
    // launch and wait for x
    if (threadIdx.x < kHRowsPerCta && blockIdx.x * kHRowsPerCta + threadIdx.x < r)
        prefetch_l2(A + (int64_t)(blockIdx.x * kHRowsPerCta + threadIdx.x) * d, (uint32_t)d);
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
    const int nch = d / 8;  // 16-B chunks of x (8 halves)
    constexpr int kMaxCh = 4;  // d <= 8192 -> <= 4 chunks per thread
    uint4 xv[kMaxCh];
    unsigned mx = 0;
#pragma unroll
    for (int i = 0; i < kMaxCh; i++) {
        const int c = threadIdx.x + i * kHThreads;
        xv[i] = c < nch ? reinterpret_cast<const uint4 *>(x)[c] : make_uint4(0, 0, 0, 0);
        const unsigned m2 = __vmaxu2(__vmaxu2(xv[i].x & 0x7fff7fffu, xv[i].y & 0x7fff7fffu),
                                     __vmaxu2(xv[i].z & 0x7fff7fffu, xv[i].w & 0x7fff7fffu));
        mx = max(mx, max(m2 & 0xffffu, m2 >> 16));
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) red_u[warp] = mx;
    __syncthreads();
    mx = red_u[0];
#pragma unroll
    for (int w = 1; w < kHThreads / 32; w++) mx = max(mx, red_u[w]);
    if (mx >= 0x7c00) {  // Inf / NaN input: flag and quantise as zero
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(err, 1u);
        mx = 0;
    }
    const float M = __half2float(__ushort_as_half((unsigned short)mx));
    const float inv = mx ? 127.f / M : 0.f;
#pragma unroll
    for (int i = 0; i < kMaxCh; i++) {
        const int c = threadIdx.x + i * kHThreads;
        if (c >= nch) break;
        const uint32_t w[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
        uint32_t packed[2] = {0, 0};
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const unsigned short b = (unsigned short)(w[e >> 1] >> (16 * (e & 1)));
            int q = 0;
            if (mx) {
                q = q127_f32(__half2float(__ushort_as_half((unsigned short)(b & 0x7fff))), M, inv);
                if (b & 0x8000) q = -q;
            }
            packed[e >> 2] |= (uint32_t)(q & 0xff) << (8 * (e & 3));
        }
        reinterpret_cast<uint2 *>(xq)[c] = make_uint2(packed[0], packed[1]);
    }
    __syncthreads();
    // dot: warps [4 rr, 4 rr + 4) handle row rr, each a quarter of d
    const int wpr = (kHThreads / 32) / kHRowsPerCta;
    const int rr = warp / wpr, seg = warp % wpr;
    const int row = blockIdx.x * kHRowsPerCta + rr;
    const int n16 = d / 16, per = (n16 + wpr - 1) / wpr;
    const int c0 = seg * per, c1 = min(n16, c0 + per);
    int acc = 0;
    if (row < r) {
        const int4 *a4 = reinterpret_cast<const int4 *>(A + (int64_t)row * d);
        const int4 *x4 = reinterpret_cast<const int4 *>(xq);
        for (int c = c0 + lane; c < c1; c += 32) {
            const int4 av = __ldg(a4 + c);
            const int4 xv4 = x4[c];
            acc = __dp4a(av.x, xv4.x, acc);
            acc = __dp4a(av.y, xv4.y, acc);
            acc = __dp4a(av.z, xv4.z, acc);
            acc = __dp4a(av.w, xv4.w, acc);
        }
    }
    acc = warp_sum_i(acc);
    if (lane == 0) red_i[warp] = acc;
    __syncthreads();
    if (threadIdx.x < kHRowsPerCta) {
        const int rw = blockIdx.x * kHRowsPerCta + threadIdx.x;
        int s = 0;
        for (int w = 0; w < wpr; w++) s += red_i[threadIdx.x * wpr + w];
        if (rw < r) h[rw] = s;
    }
}

// a2: hq = Q(h) (every CTA, redundantly), s = B hq for this CTA's rows; LPR lanes per row.
// Decode path: also the 4096-bin histogram of (s + smax) >> sh for the select kernel.
template <int LPR>
__global__ void __launch_bounds__(kSThreads) k_pred_s(int r, int F_r, int rows_per_cta,
                                                      const int32_t *__restrict__ h,
                                                      const int8_t *__restrict__ B,
                                                      int32_t *__restrict__ s, int *__restrict__ hist,
                                                      int smax, int sh) {
    __shared__ __align__(16) int8_t hq[512];
    __shared__ int red[kSThreads / 32];
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
    int mh = 0;
    for (int i = threadIdx.x; i < r; i += kSThreads) mh = max(mh, abs(h[i]));
    mh = __reduce_max_sync(0xffffffffu, (unsigned)mh);
    if (lane == 0) red[warp] = mh;
    __syncthreads();
    mh = red[0];
#pragma unroll
    for (int w = 1; w < kSThreads / 32; w++) mh = max(mh, red[w]);
    const double Mh = (double)mh, invh = mh ? 127.0 / Mh : 0.0;
    for (int i = threadIdx.x; i < r; i += kSThreads) {
        const int hv = h[i];
        int q = mh ? q127_f64((double)abs(hv), Mh, invh) : 0;
        hq[i] = (int8_t)(hv < 0 ? -q : q);
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
    cudaError_t e = launch_k(k_pred_h, dim3((r + kHRowsPerCta - 1) / kHRowsPerCta),
                             dim3(kHThreads), (size_t)d, st, d, r, x, L.A, c->ws.h, c->ws.err, pf);
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

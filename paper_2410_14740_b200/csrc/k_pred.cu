// k_pred.cu -- a1/a2: the low-rank neuron-score predictor.
//
// Paper: "A low-rank predictor locates the necessary neurons" (P:73 step 1), one predictor per
// layer driven by the layer's input, assigning "a predicted score to each neuron"
// (Deja Vu).  Form and precision are unspecified; R2: s = B * Q(A * Q(x))
// with INT8 factors and exact integer arithmetic (dp4a, int32 accumulation), so scores are
// bit-identical for any reduction order.  The requantisations use an fp32 estimate pinned to
// the exact integer result by two int64 checks (quant127_est).
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kHRowsPerCta = 2;    // rows of A per CTA (8 warps per row)
constexpr int kHThreads = 512;
constexpr int kSRowsPerCta = 64;   // rows of B per CTA

// x fp16 value -> exact integer X = x * 2^24 (every fp16 is a multiple of 2^-24).
__device__ __forceinline__ long long half_bits_to_X(unsigned short b) {
    const int e = (b >> 10) & 0x1f, m = b & 0x3ff;
    long long mag = (e == 0) ? (long long)m : ((long long)(1024 + m) << (e - 1));
    return (b & 0x8000) ? -mag : mag;
}

// a1: xq = Q(x) (every CTA, redundantly: d <= 8K halves from L2), h = A xq for 2 rows.
__global__ void __launch_bounds__(kHThreads) k_pred_h(int d, int r, const __half *__restrict__ x,
                                                      const int8_t *__restrict__ A,
                                                      int32_t *__restrict__ h, uint32_t *err) {
    extern __shared__ __align__(16) int8_t xq[];
    __shared__ unsigned red_u[kHThreads / 32];
    __shared__ int red_i[kHThreads / 32];
    // independent of the predecessor: pull this CTA's rows of A towards L2, let the next
    // kernel launch, then wait for x
    if (threadIdx.x < kHRowsPerCta && blockIdx.x * kHRowsPerCta + threadIdx.x < r)
        prefetch_l2(A + (int64_t)(blockIdx.x * kHRowsPerCta + threadIdx.x) * d, (uint32_t)d);
    griddep_launch();
    griddep_wait();
    const unsigned short *xb = reinterpret_cast<const unsigned short *>(x);
    unsigned mx = 0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) mx = max(mx, (unsigned)(xb[j] & 0x7fff));
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) red_u[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) mx = max(mx, red_u[w]);
    if (mx >= 0x7c00) {  // Inf / NaN input: flag and quantise as zero
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(err, 1u);
        mx = 0;
    }
    const long long M = half_bits_to_X((unsigned short)mx);
    const float inv = mx ? 127.f / __half2float(__ushort_as_half((unsigned short)mx)) : 0.f;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        const unsigned short b = xb[j];
        const float est = fabsf(__half2float(__ushort_as_half(b))) * inv + 0.5f;
        xq[j] = (mx == 0) ? 0 : (int8_t)quant127_est(half_bits_to_X(b), M, est);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpr = (kHThreads / 32) / kHRowsPerCta;  // warps per row
    const int rr = warp / wpr, seg = warp % wpr;
    const int row = blockIdx.x * kHRowsPerCta + rr;
    const int nchunk = d / 16, per = (nchunk + wpr - 1) / wpr;
    const int c0 = seg * per, c1 = min(nchunk, c0 + per);
    int acc = 0;
    if (row < r) {
        const int4 *a4 = reinterpret_cast<const int4 *>(A + (int64_t)row * d);
        const int4 *x4 = reinterpret_cast<const int4 *>(xq);
        for (int c = c0 + lane; c < c1; c += 32) {
            const int4 av = __ldg(a4 + c);
            const int4 xv = x4[c];
            acc = __dp4a(av.x, xv.x, acc);
            acc = __dp4a(av.y, xv.y, acc);
            acc = __dp4a(av.z, xv.z, acc);
            acc = __dp4a(av.w, xv.w, acc);
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

// a2: hq = Q(h) (every CTA, redundantly), s = B hq for 64 rows.  LPR lanes per row of B.
template <int LPR>
__global__ void __launch_bounds__(256) k_pred_s(int r, int F_r, const int32_t *__restrict__ h,
                                                const int8_t *__restrict__ B,
                                                int32_t *__restrict__ s, int *__restrict__ hist,
                                                int smax, int sh) {
    __shared__ __align__(16) int8_t hq[512];
    __shared__ int red[8];
    if (threadIdx.x == 0) {  // this CTA's 64 rows of B are contiguous
        const int base = blockIdx.x * kSRowsPerCta;
        const int rows = min(kSRowsPerCta, F_r - base);
        if (rows > 0) prefetch_l2(B + (int64_t)base * r, (uint32_t)(rows * r));
    }
    griddep_launch();
    griddep_wait();
    int mh = 0;
    for (int i = threadIdx.x; i < r; i += blockDim.x) mh = max(mh, abs(h[i]));
    mh = __reduce_max_sync(0xffffffffu, (unsigned)mh);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mh;
    __syncthreads();
    mh = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) mh = max(mh, red[w]);
    const float inv = mh ? 127.f / (float)mh : 0.f;
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
        const int hv = h[i];
        hq[i] = (int8_t)quant127_est(hv, mh, fabsf((float)hv) * inv + 0.5f);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int RPW = 32 / LPR;  // rows per warp iteration
    const int part = lane % LPR, sub = lane / LPR;
    const int4 hv = reinterpret_cast<const int4 *>(hq)[part];
    const int base = blockIdx.x * kSRowsPerCta;
    for (int rr = warp * RPW; rr < kSRowsPerCta; rr += 8 * RPW) {
        const int row = base + rr + sub;
        int acc = 0;
        if (row < F_r) {
            const int4 bv = __ldg(reinterpret_cast<const int4 *>(B + (int64_t)row * r) + part);
            acc = __dp4a(bv.x, hv.x, acc);
            acc = __dp4a(bv.y, hv.y, acc);
            acc = __dp4a(bv.z, hv.z, acc);
            acc = __dp4a(bv.w, hv.w, acc);
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (part == 0 && row < F_r) {
            s[row] = acc;
            // decode path: 4096-bin histogram of (s + smax) >> sh for the fused select
            if (hist) atomicAdd(&hist[(acc + smax) >> sh], 1);
        }
    }
}

}  // namespace

cudaError_t launch_predict(m2c_ctx *c, const LayerState &L, const __half *x, int32_t *scores,
                           int *hist, cudaStream_t st) {
    const int d = c->desc.d_model, r = c->desc.pred_rank, F_r = c->F_r;
    cudaError_t e = launch_k(k_pred_h, dim3((r + kHRowsPerCta - 1) / kHRowsPerCta),
                             dim3(kHThreads), (size_t)d, st, d, r, x, L.A, c->ws.h, c->ws.err);
    if (e != cudaSuccess) return e;
    c->launch_counter++;
    const dim3 grid((F_r + kSRowsPerCta - 1) / kSRowsPerCta), block(256);
    const int sm = c->sel_smax, sh = c->sel_sh;
    switch (r / 16) {
        case 1: e = launch_k(k_pred_s<1>, grid, block, 0, st, r, F_r, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 2: e = launch_k(k_pred_s<2>, grid, block, 0, st, r, F_r, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 4: e = launch_k(k_pred_s<4>, grid, block, 0, st, r, F_r, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 8: e = launch_k(k_pred_s<8>, grid, block, 0, st, r, F_r, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 16: e = launch_k(k_pred_s<16>, grid, block, 0, st, r, F_r, c->ws.h, L.B, scores, hist, sm, sh); break;
        case 32: e = launch_k(k_pred_s<32>, grid, block, 0, st, r, F_r, c->ws.h, L.B, scores, hist, sm, sh); break;
        default: return cudaErrorInvalidValue;
    }
    c->launch_counter++;
    return e;
}

}  // namespace m2c

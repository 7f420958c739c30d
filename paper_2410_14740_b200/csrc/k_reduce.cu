// k_reduce.cu -- a7: deterministic reduction of the per-CTA partial sums, fp16 output and the
// stack residual x_{l+1} = fp16(x_l + fp16(y_l)) (R14), plus small helpers.
// The reduction order is fixed (partial rows in ascending order within each of 8 warp lanes,
// then the 8 lanes in order), so y is bit-reproducible run to run.
#include "m2c_internal.cuh"

namespace m2c {
namespace {

// grid d/32 CTAs x 1024 threads: lane = element of a 32-element slice, warp w sums rows w::32
// (<= 10 independent loads in flight per thread), then warp 0 sums the 32 warp totals.
__global__ void __launch_bounds__(1024) k_reduce(int d, int np, const float *__restrict__ partial,
                                                 const __half *x, float *__restrict__ y32,
                                                 __half *__restrict__ y16, __half *x_next,
                                                 int *__restrict__ hist_zero, const int8_t *__restrict__ At_next,
                                                 long long *__restrict__ h_next, int r, uint32_t *__restrict__ err) {
    __shared__ float sm[32][33];
    __shared__ int xm[32], xsh[32];
    griddep_launch();
    griddep_wait();
    // the FFN that read the score histogram is complete: clear it for the next layer
    if (hist_zero)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 4096; i += gridDim.x * blockDim.x)
            hist_zero[i] = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int e = blockIdx.x * 32 + lane;
    float v[10];
#pragma unroll
    for (int i = 0; i < 10; i++) {
        const int r = warp + 32 * i;
        v[i] = r < np ? partial[(int64_t)r * d + e] : 0.f;
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 10; i++) acc += v[i];
    for (int r = warp + 320; r < np; r += 32) acc += partial[(int64_t)r * d + e];
    sm[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
        float y = 0.f;
#pragma unroll
        for (int w = 0; w < 32; w++) y += sm[w][lane];
        if (y32) y32[e] = y;
        const __half yh = __float2half_rn(y);
        if (y16) y16[e] = yh;
        const __half xn = __hadd(x[e], yh);  // (x_next may alias x)
        if (x_next) x_next[e] = xn;
        if (At_next) {  // the next layer's h = A x: this chunk's exact integer part (R2)
            bool bad = false;
            int m, sh;
            fp16_fixed(__half_as_ushort(xn), m, sh, bad);
            if (bad) flag_error(err, 1u);
            xm[lane] = m;
            xsh[lane] = sh;
        }
    }
    if (At_next) {  // (LRU engine: the next layer's select-only k_decode skips its prologue)
        __syncthreads();
        const int8_t *A = At_next + (int64_t)blockIdx.x * 32 * r;  // the chunk's 32 rows of A^T
        for (int i2 = threadIdx.x; i2 < 2 * r; i2 += blockDim.x) {
            const int i = i2 >> 1, j0 = 16 * (i2 & 1);
            unsigned long long acc = 0;
#pragma unroll
            for (int j = 0; j < 16; j++)
                acc += (unsigned long long)(long long)((int)A[(int64_t)(j0 + j) * r + i] * xm[j0 + j]) << xsh[j0 + j];
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            if ((i2 & 1) == 0 && acc) red_add_u64(h_next + (int64_t)i * kHStride, (long long)acc);
        }
    }
}

__global__ void k_finalize(int d, const float *__restrict__ y32, const __half *__restrict__ x,
                           __half *__restrict__ y16, __half *__restrict__ x_next) {
    griddep_wait();
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < d) {
        const __half yh = __float2half_rn(y32[e]);
        if (y16) y16[e] = yh;
        if (x_next) x_next[e] = __hadd(x[e], yh);
    }
}

__global__ void k_fill_i32(int32_t *p, int32_t v, int64_t n) {
    griddep_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_iota(int32_t *p, int64_t n) {
    griddep_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

__global__ void k_set_counts(int32_t *dst, int32_t a, int32_t b, int32_t c) {
    griddep_wait();
    dst[0] = a;
    dst[1] = b;
    dst[2] = c;
}

}  // namespace

cudaError_t launch_reduce(m2c_ctx *c, int n_partials, const float *partial, const __half *x,
                          float *y32, __half *y16, __half *x_next, int *hist_zero,
                          cudaStream_t st, const int8_t *At_next) {
    const int d = c->desc.d_model;
    cudaError_t e = launch_k(k_reduce, dim3(d / 32), dim3(1024), 0, st, d, n_partials, partial, x,
                             y32, y16, x_next, hist_zero, At_next, At_next ? c->dec_hb : (long long *)nullptr,
                             c->desc.pred_rank, c->ws.err);
    c->launch_counter++;
    return e;
}

cudaError_t launch_finalize(m2c_ctx *c, const float *y32, const __half *x, __half *y16,
                            __half *x_next, cudaStream_t st) {
    const int d = c->desc.d_model;
    cudaError_t e = launch_k(k_finalize, dim3((d + 255) / 256), dim3(256), 0, st, d, y32, x, y16,
                             x_next);
    c->launch_counter++;
    return e;
}

cudaError_t launch_fill_i32(int32_t *p, int32_t v, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    return launch_k(k_fill_i32, dim3((unsigned)blocks), dim3(256), 0, st, p, v, n);
}

cudaError_t launch_iota(int32_t *p, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    return launch_k(k_iota, dim3((unsigned)blocks), dim3(256), 0, st, p, n);
}

cudaError_t launch_set_counts(int32_t *dst, int32_t a, int32_t b, int32_t c, cudaStream_t st) {
    return launch_k(k_set_counts, dim3(1), dim3(1), 0, st, dst, a, b, c);
}

}  // namespace m2c

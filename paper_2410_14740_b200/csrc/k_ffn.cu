// k_ffn.cu -- a6: fused dequant-GEMV (gate, up) -> act(g) * u -> sparse down-projection.
//
// Paper: a neuron is a row of the first FFN matrices and the matching column of the next
// (P:58); only the active neurons are computed; the cache unit memory "can be
// directly used for inference computation, avoiding unnecessary copying from the cache to
// inference tensors"; low-bit neurons are dequantised for compute.  Decode is
// memory-bound: batch-1 GEMV at ~1 flop/byte, so CUDA cores, not tensor cores.
//
// B200 design: a persistent grid (one CTA per SM).  Each CTA owns a contiguous, byte-balanced
// share of the active records (tier order FP16, INT8, INT4).  One elected thread streams the
// records into a shared-memory byte ring with 1-D TMA bulk copies (cp.async.bulk, SASS
// UBLKCP) completing on per-record mbarriers; every thread owns the same 16 (or 8) elements
// of d for gate, up, down and x, so the down-projection accumulates in registers.  g and u
// are reduced per batch of records with warp shuffles + one smem round.  Dequant is
// in-register: per 128-group s * (sum q x - z sum x) (R5).  The per-CTA partial y
// goes to a [G][d] fp32 buffer reduced deterministically by k_reduce.
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kNB = 4;          // records per reduction batch
constexpr int kNSlot = 32;      // mbarriers in the ring
constexpr int kRingBytes = 200 * 1024;  // 1 CTA per SM; + ~9 KB static

struct FfnArgs {
    const uint8_t *pool[3];
    int64_t nb[3];
    int seg[3];
    int w16[3];  // record size in 16-B units (byte-balancing weights)
};

__device__ __forceinline__ float q2f(uint32_t q) {  // exact small unsigned int -> float
    return __uint_as_float(0x4B000000u | q) - 8388608.0f;
}

template <int NCH>
struct Acc {
    float y[NCH][8];
    float bias[NCH];
};

// x chunk helpers
template <int NCH>
__device__ __forceinline__ void load_x(const __half *x, int T, float (&xf)[NCH][8],
                                       float (&xs)[NCH]) {
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        const int q = c * T + threadIdx.x;
        const uint4 raw = *reinterpret_cast<const uint4 *>(x + 8 * q);
        const __half2 *h = reinterpret_cast<const __half2 *>(&raw);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float2 f = __half22float2(h[i]);
            xf[c][2 * i] = f.x;
            xf[c][2 * i + 1] = f.y;
            s += f.x + f.y;
        }
        xs[c] = s;
    }
}

// gate/up partial dot products of this thread's chunks for one record in smem
template <int NCH>
__device__ __forceinline__ void dot_gu(int tier, const uint8_t *rec, int d, int T,
                                       const float (&xf)[NCH][8], const float (&xs)[NCH],
                                       float &pg, float &pu) {
    pg = 0.f;
    pu = 0.f;
    const int G = d >> 7;
    if (tier == 0) {
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            const int q = c * T + threadIdx.x;
#pragma unroll
            for (int m = 0; m < 2; m++) {
                const uint4 raw = *reinterpret_cast<const uint4 *>(rec + (size_t)m * 2 * d + 16 * q);
                const __half2 *h = reinterpret_cast<const __half2 *>(&raw);
                float acc = 0.f;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const float2 f = __half22float2(h[i]);
                    acc = fmaf(f.x, xf[c][2 * i], acc);
                    acc = fmaf(f.y, xf[c][2 * i + 1], acc);
                }
                if (m == 0) pg += acc; else pu += acc;
            }
        }
    } else if (tier == 1) {
        const uint8_t *scales = rec + 3 * d;
        const uint8_t *zeros = scales + 6 * G;
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            const int q = c * T + threadIdx.x;
            const int grp = q >> 4;
#pragma unroll
            for (int m = 0; m < 2; m++) {
                const uint2 raw = *reinterpret_cast<const uint2 *>(rec + (size_t)m * d + 8 * q);
                float acc = 0.f;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    acc = fmaf(q2f(__byte_perm(raw.x, 0, 0x4440 | i)), xf[c][i], acc);
                    acc = fmaf(q2f(__byte_perm(raw.y, 0, 0x4440 | i)), xf[c][4 + i], acc);
                }
                const float s = __half2float(*reinterpret_cast<const __half *>(scales + 2 * (m * G + grp)));
                const float z = (float)zeros[m * G + grp];
                const float v = s * fmaf(-z, xs[c], acc);
                if (m == 0) pg += v; else pu += v;
            }
        }
    } else {
        const uint8_t *scales = rec + 3 * (d >> 1);
        const uint8_t *zeros = scales + 6 * G;
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            const int q = c * T + threadIdx.x;
            const int grp = q >> 4;
#pragma unroll
            for (int m = 0; m < 2; m++) {
                const uint32_t w = *reinterpret_cast<const uint32_t *>(rec + (size_t)m * (d >> 1) + 4 * q);
                float acc = 0.f;
#pragma unroll
                for (int i = 0; i < 8; i++) acc = fmaf(q2f((w >> (4 * i)) & 0xFu), xf[c][i], acc);
                const float s = __half2float(*reinterpret_cast<const __half *>(scales + 2 * (m * G + grp)));
                const float z = (float)zeros[m * G + grp];
                const float v = s * fmaf(-z, xs[c], acc);
                if (m == 0) pg += v; else pu += v;
            }
        }
    }
}

// y += a * deq(down column) for this thread's chunks
template <int NCH>
__device__ __forceinline__ void axpy_down(int tier, const uint8_t *rec, int d, int T, float a,
                                          Acc<NCH> &acc) {
    const int G = d >> 7;
    if (tier == 0) {
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            const int q = c * T + threadIdx.x;
            const uint4 raw = *reinterpret_cast<const uint4 *>(rec + (size_t)4 * d + 16 * q);
            const __half2 *h = reinterpret_cast<const __half2 *>(&raw);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const float2 f = __half22float2(h[i]);
                acc.y[c][2 * i] = fmaf(a, f.x, acc.y[c][2 * i]);
                acc.y[c][2 * i + 1] = fmaf(a, f.y, acc.y[c][2 * i + 1]);
            }
        }
    } else if (tier == 1) {
        const uint8_t *scales = rec + 3 * d;
        const uint8_t *zeros = scales + 6 * G;
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            const int q = c * T + threadIdx.x;
            const int grp = q >> 4;
            const uint2 raw = *reinterpret_cast<const uint2 *>(rec + (size_t)2 * d + 8 * q);
            const float as = a * __half2float(*reinterpret_cast<const __half *>(scales + 2 * (2 * G + grp)));
            acc.bias[c] = fmaf(-as, (float)zeros[2 * G + grp], acc.bias[c]);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                acc.y[c][i] = fmaf(as, q2f(__byte_perm(raw.x, 0, 0x4440 | i)), acc.y[c][i]);
                acc.y[c][4 + i] = fmaf(as, q2f(__byte_perm(raw.y, 0, 0x4440 | i)), acc.y[c][4 + i]);
            }
        }
    } else {
        const uint8_t *scales = rec + 3 * (d >> 1);
        const uint8_t *zeros = scales + 6 * G;
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            const int q = c * T + threadIdx.x;
            const int grp = q >> 4;
            const uint32_t w = *reinterpret_cast<const uint32_t *>(rec + (size_t)d + 4 * q);
            const float as = a * __half2float(*reinterpret_cast<const __half *>(scales + 2 * (2 * G + grp)));
            acc.bias[c] = fmaf(-as, (float)zeros[2 * G + grp], acc.bias[c]);
#pragma unroll
            for (int i = 0; i < 8; i++) acc.y[c][i] = fmaf(as, q2f((w >> (4 * i)) & 0xFu), acc.y[c][i]);
        }
    }
}

template <int NCH>
__global__ void __launch_bounds__(NCH == 2 ? 512 : 1024, 1)
    k_ffn(FfnArgs a, int d, int act, const __half *__restrict__ x,
          const int32_t *__restrict__ items, const int32_t *__restrict__ counts,
          float *__restrict__ partial, int nbmax) {
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ __align__(8) uint64_t bars[kNSlot];
    __shared__ float red[32][kNB][2];
    const int T = blockDim.x;
    const int nwarp = T >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kNSlot; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    griddep_wait();

    // ---- this CTA's byte-balanced share of the records ----
    int n_t[3], i_lo[3], i_hi[3];
    long long W = 0, base[3];
    for (int t = 0; t < 3; t++) {
        n_t[t] = counts[t];
        base[t] = W;
        W += (long long)n_t[t] * a.w16[t];
    }
    const long long lo = W * blockIdx.x / gridDim.x, hi = W * (blockIdx.x + 1) / gridDim.x;
    int n_items = 0;
    for (int t = 0; t < 3; t++) {
        const long long w = a.w16[t];
        long long s0 = lo - base[t], s1 = hi - base[t];
        s0 = s0 <= 0 ? 0 : (s0 + w - 1) / w;
        s1 = s1 <= 0 ? 0 : (s1 + w - 1) / w;
        i_lo[t] = (int)min((long long)n_t[t], s0);
        i_hi[t] = (int)min((long long)n_t[t], s1);
        n_items += i_hi[t] - i_lo[t];
    }
    const int c1 = i_hi[0] - i_lo[0], c2 = c1 + i_hi[1] - i_lo[1];
    auto tier_of_j = [&](int j) { return j < c1 ? 0 : (j < c2 ? 1 : 2); };
    auto src_of_j = [&](int j, int t) -> const uint8_t * {
        const int i = i_lo[t] + j - (t == 0 ? 0 : (t == 1 ? c1 : c2));
        const int slot = items[a.seg[t] + i];
        return a.pool[t] + (int64_t)slot * a.nb[t];
    };

    // ---- producer state (thread 0 only) ----
    int issued = 0;
    long long v_issue = 0;          // virtual end of the last issued record
    long long v_cons = 0;           // virtual start of the oldest unconsumed record
    const uint64_t pol = policy_evict_first();
    auto issue_more = [&](int consumed) {
        while (issued < n_items && issued - consumed < kNSlot) {
            const int t = tier_of_j(issued);
            const long long sz = a.nb[t];
            long long v = v_issue;
            if ((v % kRingBytes) + sz > kRingBytes) v = (v / kRingBytes + 1) * kRingBytes;
            if (v + sz - v_cons > kRingBytes) break;
            uint64_t *bar = &bars[issued % kNSlot];
            mbar_expect_tx(bar, (uint32_t)sz);
            bulk_g2s(ring + (v % kRingBytes), src_of_j(issued, t), (uint32_t)sz, bar, pol);
            v_issue = v + sz;
            issued++;
        }
    };
    if (threadIdx.x == 0) issue_more(0);

    float xf[NCH][8], xs[NCH];
    load_x<NCH>(x, T, xf, xs);
    Acc<NCH> acc;
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        acc.bias[c] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; i++) acc.y[c][i] = 0.f;
    }

    long long v_next = 0;  // consumer-side virtual cursor (identical sequence in every thread)
    for (int j0 = 0; j0 < n_items; j0 += nbmax) {
        const int nbatch = min(nbmax, n_items - j0);
        int off[kNB], tr[kNB];
        long long vstart0 = 0;
#pragma unroll
        for (int b = 0; b < kNB; b++) {
            if (b < nbatch) {
                const int j = j0 + b;
                tr[b] = tier_of_j(j);
                const long long sz = a.nb[tr[b]];
                long long v = v_next;
                if ((v % kRingBytes) + sz > kRingBytes) v = (v / kRingBytes + 1) * kRingBytes;
                if (b == 0) vstart0 = v;
                off[b] = (int)(v % kRingBytes);
                v_next = v + sz;
                mbar_wait(&bars[j % kNSlot], (uint32_t)((j / kNSlot) & 1));
            }
        }
        float pg[kNB], pu[kNB];
#pragma unroll
        for (int b = 0; b < kNB; b++) {
            pg[b] = 0.f;
            pu[b] = 0.f;
            if (b < nbatch) dot_gu<NCH>(tr[b], ring + off[b], d, T, xf, xs, pg[b], pu[b]);
        }
#pragma unroll
        for (int b = 0; b < kNB; b++) {
            pg[b] = warp_sum_f(pg[b]);
            pu[b] = warp_sum_f(pu[b]);
        }
        if (lane == 0) {
#pragma unroll
            for (int b = 0; b < kNB; b++) {
                red[warp][b][0] = pg[b];
                red[warp][b][1] = pu[b];
            }
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < kNB; b++) {
            if (b < nbatch) {
                float g = 0.f, u = 0.f;
                for (int w = 0; w < nwarp; w++) {
                    g += red[w][b][0];
                    u += red[w][b][1];
                }
                const float av = (act == 1) ? fmaxf(g, 0.f) * u : g / (1.f + expf(-g)) * u;
                axpy_down<NCH>(tr[b], ring + off[b], d, T, av, acc);
            }
        }
        __syncthreads();  // records of this batch fully consumed; red[] reusable
        if (threadIdx.x == 0) {
            v_cons = v_next;  // everything up to the end of this batch is free
            (void)vstart0;
            fence_proxy_async();
            issue_more(j0 + nbatch);
        }
    }
    griddep_launch();
    // ---- partial y of this CTA ----
    float *out = partial + (int64_t)blockIdx.x * d;
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        const int q = c * T + threadIdx.x;
        float4 v0, v1;
        v0.x = acc.y[c][0] + acc.bias[c];
        v0.y = acc.y[c][1] + acc.bias[c];
        v0.z = acc.y[c][2] + acc.bias[c];
        v0.w = acc.y[c][3] + acc.bias[c];
        v1.x = acc.y[c][4] + acc.bias[c];
        v1.y = acc.y[c][5] + acc.bias[c];
        v1.z = acc.y[c][6] + acc.bias[c];
        v1.w = acc.y[c][7] + acc.bias[c];
        reinterpret_cast<float4 *>(out + 8 * q)[0] = v0;
        reinterpret_cast<float4 *>(out + 8 * q)[1] = v1;
    }
}

}  // namespace

cudaError_t init_ffn_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_ffn<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_ffn<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
    return e;
}

int ffn_nch(int d) { return (d % 512 == 0 && d >= 1024) ? 2 : 1; }

cudaError_t launch_ffn(m2c_ctx *c, const LayerState &L, const __half *x, const int32_t *items,
                       const int32_t *counts, const m2c_tier_plan &p, float *partial,
                       cudaStream_t st) {
    const int d = c->desc.d_model;
    FfnArgs a;
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8};
    for (int t = 0; t < 3; t++) {
        a.pool[t] = L.pool[t];
        a.nb[t] = c->nb[t];
        a.seg[t] = seg[t];
        a.w16[t] = (int)(c->nb[t] / 16);
    }
    const int nch = ffn_nch(d);
    const int T = d / (8 * nch);
    const size_t smem = kRingBytes;
    // a batch must fit in the ring even after a wrap: nbmax * nb16 + nb16 <= ring
    int nbmax = (int)(kRingBytes / c->nb[0]) - 1;
    nbmax = nbmax < 1 ? 1 : (nbmax > kNB ? kNB : nbmax);
    cudaError_t e;
    if (nch == 2) {
        e = launch_k(k_ffn<2>, dim3(c->G), dim3(T), smem, st, a, d, c->desc.act, x, items,
                         counts, partial, nbmax);
    } else {
        e = launch_k(k_ffn<1>, dim3(c->G), dim3(T), smem, st, a, d, c->desc.act, x, items,
                         counts, partial, nbmax);
    }
    c->launch_counter++;
    return e;
}

}  // namespace m2c

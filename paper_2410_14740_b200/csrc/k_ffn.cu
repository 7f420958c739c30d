// k_ffn.cu -- a6: fused dequant-GEMV (gate, up) -> act(g) * u -> sparse down-projection,
// and (decode path) the fused top-k/tier split in front of it.
//
// Paper: a neuron is a row of the first FFN matrices and the matching column of the next
// (P:58); only the active neurons are computed; the cache unit memory "can be
// directly used for inference computation, avoiding unnecessary copying from the cache to
// inference tensors"; low-bit neurons are dequantised for compute.  Decode is
// memory-bound: batch-1 GEMV at ~1 flop/byte, so CUDA cores, not tensor cores.
//
// B200 design (one persistent CTA per SM, T = d/8 threads):
//  * Work split: each CTA owns a contiguous share of the active records (tier order FP16,
//    INT8, INT4), balanced on bytes + lambda * weights (memory and issue cost both matter:
//    an INT4 record has 1/4 of the bytes of an FP16 one but the same 3d weights to dequant).
//  * Records stream into a shared-memory byte ring by 1-D TMA bulk copies (cp.async.bulk,
//    SASS UBLKCP), one mbarrier per record, issued by one thread as ring space frees.
//  * Batches of up to 16 records: gate/up dot products are warp-local (one warp, or a few
//    warps splitting d, per record; warp-shuffle reductions only), then one barrier, then the
//    down-projection where thread t owns elements [8t, 8t+8) of y in registers.
//  * Dequant in registers, ~2 instructions per weight: codes become the fp16 value 1024 + q
//    (or 1024 + 16q for odd INT4 nibbles) by PRMT/LOP3 (magic-exponent trick); HFMA2 removes
//    the offset and zero point exactly; fma.rn.f32.f16 (SASS FHFMA) multiplies exact fp16
//    (q - z) by fp16 x with an exact product and fp32 accumulation.  Per 128-group
//    s * sum (q - z) x (R5).
//  * The per-CTA partial y goes to a [G][d] fp32 buffer reduced in a fixed order by k_reduce.
//  * k_ffn_sel (decode path) first derives the FP16/INT8/INT4 tier lists itself, redundantly
//    in every CTA, from the predictor scores and the 4096-bin score histogram k_pred_s left in
//    global memory (exact thresholds via a second-level histogram, ties by ascending id),
//    and before waiting on its predecessor prefetches into L2 the records the previous token
//    selected for this layer (~80% of them recur).
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kNBMax = 16;   // records per batch
constexpr int kNSlot = 32;   // mbarriers (>= records in flight)
constexpr int kRingList = 192 * 1024;  // == kRingSel: identical batching, bit-identical y
constexpr int kRingSel = 192 * 1024;
constexpr int kHistBins = 4096;
constexpr int kMaxLocal = 1024;  // records one CTA may own

struct FfnArgs {
    const uint8_t *pool[3];
    int nb[3];     // record bytes per tier
    int seg[3];    // tier segment offsets in the item lists
    int wt[3];     // balancing weight per record (bytes + lambda * 3d), in 16-B units
};

struct SelArgs {
    const int32_t *scores;  // [F_r]
    const int32_t *hist;    // [4096] histogram of (s + smax) >> sh
    int32_t *out_ids;       // [k] tier lists written by CTA 0 (also next token's prefetch hint)
    const int32_t *prev_ids;  // [k] previous token's lists for this layer (prefetch hint)
    int F_r, k, k16, k8, smax, sh;
};

__device__ __forceinline__ void hfma32(float &acc, uint32_t a, uint32_t b, int ha, int hb) {
    // acc += a.h[ha] * b.h[hb]  (fp16 x fp16 exact, fp32 accumulate)
    const uint16_t x = ha ? (uint16_t)(a >> 16) : (uint16_t)a;
    const uint16_t y = hb ? (uint16_t)(b >> 16) : (uint16_t)b;
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(x), "h"(y));
}
__device__ __forceinline__ float h2f_lo(uint32_t v) { return __half2float(__ushort_as_half((uint16_t)v)); }
__device__ __forceinline__ float h2f_hi(uint32_t v) { return __half2float(__ushort_as_half((uint16_t)(v >> 16))); }
__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
    const __half2 r = __hsub2(*reinterpret_cast<const __half2 *>(&a), *reinterpret_cast<const __half2 *>(&b));
    return *reinterpret_cast<const uint32_t *>(&r);
}
__device__ __forceinline__ uint32_t lop_andor(uint32_t a, uint32_t m, uint32_t c) {
    uint32_t r;  // (a & m) | c in one LOP3 with register operands
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(m), "r"(c));
    return r;
}
__device__ __forceinline__ float half_bits_f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// ---- INT8: 8 codes (2 words) -> 4 words of fp16 pairs (q - z) --------------------------
__device__ __forceinline__ void deq8(uint32_t w0, uint32_t w1, uint32_t zz, uint32_t (&p)[4]) {
    p[0] = hsub2(__byte_perm(w0, 0x64646464u, 0x4140), zz);  // elements 0, 1
    p[1] = hsub2(__byte_perm(w0, 0x64646464u, 0x4342), zz);  // 2, 3
    p[2] = hsub2(__byte_perm(w1, 0x64646464u, 0x4140), zz);  // 4, 5
    p[3] = hsub2(__byte_perm(w1, 0x64646464u, 0x4342), zz);  // 6, 7
}
// ---- INT4: 8 codes (1 word, element m in bits [4m, 4m+4)) -> 4 fp16 pairs --------------
// p[0] = (e0, e4) - z, p[1] = 16 (e1, e5) - 16 z, p[2] = (e2, e6) - z, p[3] = 16 (e3, e7) - 16 z
__device__ __forceinline__ void deq4(uint32_t w, uint32_t zz, uint32_t zz16, uint32_t (&p)[4]) {
    const uint32_t M0 = 0x000F000Fu, M1 = 0x00F000F0u, MAG = 0x64006400u;
    const uint32_t w8 = w >> 8;
    p[0] = hsub2(lop_andor(w, M0, MAG), zz);
    p[1] = hsub2(lop_andor(w, M1, MAG), zz16);
    p[2] = hsub2(lop_andor(w8, M0, MAG), zz);
    p[3] = hsub2(lop_andor(w8, M1, MAG), zz16);
}
__device__ __forceinline__ uint32_t zz2(uint32_t z) {  // fp16x2 (1024 + z)
    const uint32_t h = 0x6400u | z;
    return h | (h << 16);
}
__device__ __forceinline__ uint32_t zz2_16(uint32_t z) {  // fp16x2 (1024 + 16 z)
    const uint32_t h = 0x6400u | (z << 4);
    return h | (h << 16);
}

// ---- warp-local partial dot products of one record over chunks [c0, c1) (8 elements each)
// xs: fp16 x in smem.  Returns (gate, up) partial sums (scaled) of this lane.
template <int TIER>
__device__ __forceinline__ void gu_chunks(const uint8_t *rec, const uint4 *xs, int d, int c0, int c1,
                                          float &pg, float &pu) {
    const int lane = threadIdx.x & 31;
    const int G = d >> 7;
    float ag = 0.f, au = 0.f;
    for (int c = c0 + lane; c < c1; c += 32) {
        const uint4 xv = xs[c];
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
        if (TIER == 0) {
            const uint4 gv = *reinterpret_cast<const uint4 *>(rec + 16 * c);
            const uint4 uv = *reinterpret_cast<const uint4 *>(rec + 2 * d + 16 * c);
            const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w}, uw[4] = {uv.x, uv.y, uv.z, uv.w};
#pragma unroll
            for (int i = 0; i < 4; i++) {
                hfma32(ag, gw[i], xw[i], 0, 0);
                hfma32(ag, gw[i], xw[i], 1, 1);
                hfma32(au, uw[i], xw[i], 0, 0);
                hfma32(au, uw[i], xw[i], 1, 1);
            }
        } else {
            const uint8_t *scales = rec + (TIER == 1 ? 3 * d : 3 * (d >> 1));
            const uint8_t *zeros = scales + 6 * G;
            const int grp = c >> 4;
            const float sg = half_bits_f(*reinterpret_cast<const uint16_t *>(scales + 2 * grp));
            const float su = half_bits_f(*reinterpret_cast<const uint16_t *>(scales + 2 * (G + grp)));
            const uint32_t zg = zeros[grp], zu = zeros[G + grp];
            float tg = 0.f, tu = 0.f;
            if (TIER == 1) {
                const uint2 gv = *reinterpret_cast<const uint2 *>(rec + 8 * c);
                const uint2 uv = *reinterpret_cast<const uint2 *>(rec + d + 8 * c);
                uint32_t pg_[4], pu_[4];
                deq8(gv.x, gv.y, zz2(zg), pg_);
                deq8(uv.x, uv.y, zz2(zu), pu_);
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    hfma32(tg, pg_[i], xw[i], 0, 0);
                    hfma32(tg, pg_[i], xw[i], 1, 1);
                    hfma32(tu, pu_[i], xw[i], 0, 0);
                    hfma32(tu, pu_[i], xw[i], 1, 1);
                }
            } else {
                const uint32_t gw = *reinterpret_cast<const uint32_t *>(rec + 4 * c);
                const uint32_t uw = *reinterpret_cast<const uint32_t *>(rec + (d >> 1) + 4 * c);
                uint32_t pg_[4], pu_[4];
                deq4(gw, zz2(zg), zz2_16(zg), pg_);
                deq4(uw, zz2(zu), zz2_16(zu), pu_);
                // x pairs: (e0, e4) = (xw0.lo, xw2.lo), (e1, e5) = (xw0.hi, xw2.hi),
                //          (e2, e6) = (xw1.lo, xw3.lo), (e3, e7) = (xw1.hi, xw3.hi)
                float tg16 = 0.f, tu16 = 0.f;
                hfma32(tg, pg_[0], xw[0], 0, 0);
                hfma32(tg, pg_[0], xw[2], 1, 0);
                hfma32(tg16, pg_[1], xw[0], 0, 1);
                hfma32(tg16, pg_[1], xw[2], 1, 1);
                hfma32(tg, pg_[2], xw[1], 0, 0);
                hfma32(tg, pg_[2], xw[3], 1, 0);
                hfma32(tg16, pg_[3], xw[1], 0, 1);
                hfma32(tg16, pg_[3], xw[3], 1, 1);
                hfma32(tu, pu_[0], xw[0], 0, 0);
                hfma32(tu, pu_[0], xw[2], 1, 0);
                hfma32(tu16, pu_[1], xw[0], 0, 1);
                hfma32(tu16, pu_[1], xw[2], 1, 1);
                hfma32(tu, pu_[2], xw[1], 0, 0);
                hfma32(tu, pu_[2], xw[3], 1, 0);
                hfma32(tu16, pu_[3], xw[1], 0, 1);
                hfma32(tu16, pu_[3], xw[3], 1, 1);
                tg = fmaf(tg16, 0.0625f, tg);
                tu = fmaf(tu16, 0.0625f, tu);
            }
            ag = fmaf(sg, tg, ag);
            au = fmaf(su, tu, au);
        }
    }
    pg = ag;
    pu = au;
}

__device__ __forceinline__ void gu_any(int tier, const uint8_t *rec, const uint4 *xs, int d, int c0,
                                       int c1, float &pg, float &pu) {
    if (tier == 0) gu_chunks<0>(rec, xs, d, c0, c1, pg, pu);
    else if (tier == 1) gu_chunks<1>(rec, xs, d, c0, c1, pg, pu);
    else gu_chunks<2>(rec, xs, d, c0, c1, pg, pu);
}

// ---- y[8t .. 8t+8) += a * deq(down column) --------------------------------------------
template <int TIER>
__device__ __forceinline__ void down_t(const uint8_t *rec, int d, float a, float (&y)[8]) {
    const int t = threadIdx.x;
    if (TIER == 0) {
        const uint4 v = *reinterpret_cast<const uint4 *>(rec + 4 * d + 16 * t);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            y[2 * i] = fmaf(a, h2f_lo(w[i]), y[2 * i]);
            y[2 * i + 1] = fmaf(a, h2f_hi(w[i]), y[2 * i + 1]);
        }
    } else {
        const int G = d >> 7, grp = t >> 4;
        const uint8_t *scales = rec + (TIER == 1 ? 3 * d : 3 * (d >> 1));
        const uint32_t z = (scales + 6 * G)[2 * G + grp];
        const float as = a * half_bits_f(*reinterpret_cast<const uint16_t *>(scales + 2 * (2 * G + grp)));
        uint32_t p[4];
        if (TIER == 1) {
            const uint2 v = *reinterpret_cast<const uint2 *>(rec + 2 * d + 8 * t);
            deq8(v.x, v.y, zz2(z), p);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                y[2 * i] = fmaf(as, h2f_lo(p[i]), y[2 * i]);
                y[2 * i + 1] = fmaf(as, h2f_hi(p[i]), y[2 * i + 1]);
            }
        } else {
            const uint32_t w = *reinterpret_cast<const uint32_t *>(rec + d + 4 * t);
            deq4(w, zz2(z), zz2_16(z), p);
            const float as16 = as * 0.0625f;
            y[0] = fmaf(as, h2f_lo(p[0]), y[0]);
            y[4] = fmaf(as, h2f_hi(p[0]), y[4]);
            y[1] = fmaf(as16, h2f_lo(p[1]), y[1]);
            y[5] = fmaf(as16, h2f_hi(p[1]), y[5]);
            y[2] = fmaf(as, h2f_lo(p[2]), y[2]);
            y[6] = fmaf(as, h2f_hi(p[2]), y[6]);
            y[3] = fmaf(as16, h2f_lo(p[3]), y[3]);
            y[7] = fmaf(as16, h2f_hi(p[3]), y[7]);
        }
    }
}
__device__ __forceinline__ void down_any(int tier, const uint8_t *rec, int d, float a, float (&y)[8]) {
    if (tier == 0) down_t<0>(rec, d, a, y);
    else if (tier == 1) down_t<1>(rec, d, a, y);
    else down_t<2>(rec, d, a, y);
}

// exclusive block scan of up to 3 ints per thread; blockDim.x multiple of 32, <= 1024
__device__ __forceinline__ void block_scan3(const int v[3], int ex[3], int tot[3], int *sm /*[3][32]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
            int x = lane < nw ? sm[t * 32 + lane] : 0;
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
        tot[t] = sm[t * 32 + nw - 1];
    }
    __syncthreads();
}

// this CTA's share [i0_t, i1_t) of each tier list, balanced on wt (computed by one thread)
__device__ __forceinline__ void cta_ranges(const FfnArgs &a, int n0, int n1, int n2, int cta, int G,
                                           int (&r)[6]) {
    const long long w0 = a.wt[0], w1 = a.wt[1], w2 = a.wt[2];
    const long long W = n0 * w0 + n1 * w1 + n2 * w2;
    const long long lo = W * cta / G, hi = W * (cta + 1) / G;
    const long long base[3] = {0, n0 * w0, n0 * w0 + n1 * w1};
    const long long ww[3] = {w0, w1, w2};
    const int nn[3] = {n0, n1, n2};
#pragma unroll
    for (int t = 0; t < 3; t++) {
        long long s0 = lo - base[t], s1 = hi - base[t];
        s0 = s0 <= 0 ? 0 : (s0 + ww[t] - 1) / ww[t];
        s1 = s1 <= 0 ? 0 : (s1 + ww[t] - 1) / ww[t];
        r[2 * t] = (int)(s0 < nn[t] ? s0 : nn[t]);
        r[2 * t + 1] = (int)(s1 < nn[t] ? s1 : nn[t]);
    }
}

struct FfnShared {
    uint64_t bars[kNSlot];
    int span[kNSlot];
    float part[kNBMax][4][2];
    int rng[8];      // CTA ranges (6) + n_items, spare
    int scan[96];
    int selv[12];    // select: bins, above, value, rem ...
};

// The FFN main loop over this CTA's n_items records; item j -> (tier, global pointer)
template <int RING, class SrcFn>
__device__ __forceinline__ void ffn_loop(const FfnArgs &a, int d, int act, const __half *x, int n_items,
                                         int c1, int c2, SrcFn src, uint8_t *ring, uint4 *xs,
                                         FfnShared &sm, float *partial) {
    const int nwarp = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nbA = a.nb[0], nbB = a.nb[1], nbC = a.nb[2];
    auto size_of = [&](int j) { return j < c1 ? nbA : (j < c2 ? nbB : nbC); };
    auto tier_of = [&](int j) { return j < c1 ? 0 : (j < c2 ? 1 : 2); };
    const int nbmax_bytes = nbA > nbB ? (nbA > nbC ? nbA : nbC) : (nbB > nbC ? nbB : nbC);

    // producer state (thread 0)
    int issued = 0, pos_issue = 0, used = 0;
    const uint64_t pol = policy_evict_first();
    auto issue_more = [&](int consumed) {
        while (issued < n_items && issued - consumed < kNSlot) {
            const int j = issued;
            const int sz = size_of(j);
            const int waste = (pos_issue + sz > RING) ? RING - pos_issue : 0;
            if (used + waste + sz > RING) break;
            const int off = waste ? 0 : pos_issue;
            sm.span[j % kNSlot] = waste + sz;
            used += waste + sz;
            pos_issue = off + sz;
            uint64_t *bar = &sm.bars[j % kNSlot];
            mbar_expect_tx(bar, (uint32_t)sz);
            bulk_g2s(ring + off, src(j), (uint32_t)sz, bar, pol);
            issued++;
        }
    };
    if (threadIdx.x == 0) {
        fence_proxy_async();
        issue_more(0);
    }
    // x -> smem as fp16 (read by the warp-local dot products)
    for (int c = threadIdx.x; c < d / 8; c += blockDim.x) xs[c] = reinterpret_cast<const uint4 *>(x)[c];
    __syncthreads();

    float y[8];
#pragma unroll
    for (int i = 0; i < 8; i++) y[i] = 0.f;
    const int nchunk = d / 8;
    int pos_cons = 0;
    for (int j0 = 0; j0 < n_items;) {
        // batch: consecutive records that fit the ring together (with wrap slack)
        int nb = 0, bytes = 0;
        while (nb < kNBMax && j0 + nb < n_items && bytes + size_of(j0 + nb) + nbmax_bytes <= RING) {
            bytes += size_of(j0 + nb);
            nb++;
        }
        if (nb == 0) nb = 1;
        int offs[kNBMax];
#pragma unroll
        for (int b = 0; b < kNBMax; b++) {
            offs[b] = 0;
            if (b < nb) {
                const int sz = size_of(j0 + b);
                if (pos_cons + sz > RING) pos_cons = 0;
                offs[b] = pos_cons;
                pos_cons += sz;
            }
        }
        // gate/up: unit u = (item b, part p) per warp; P parts split the chunks of d
        const int P = nwarp / nb >= 4 ? 4 : (nwarp / nb >= 1 ? nwarp / nb : 1);
        for (int u = warp; u < nb * P; u += nwarp) {
            const int b = u % nb, p = u / nb;
            const int j = j0 + b;
            mbar_wait(&sm.bars[j % kNSlot], (uint32_t)((j / kNSlot) & 1));
            const int c0 = nchunk * p / P, c1x = nchunk * (p + 1) / P;
            float pg, pu;
            int rb = 0;
#pragma unroll
            for (int bb = 0; bb < kNBMax; bb++) rb = (bb == b) ? offs[bb] : rb;
            gu_any(tier_of(j), ring + rb, xs, d, c0, c1x, pg, pu);
            pg = warp_sum_f(pg);
            pu = warp_sum_f(pu);
            if (lane == 0) {
                sm.part[b][p][0] = pg;
                sm.part[b][p][1] = pu;
            }
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < kNBMax; b++) {
            if (b < nb) {
                const int j = j0 + b;
                float g = 0.f, u = 0.f;
                for (int p = 0; p < P; p++) {
                    g += sm.part[b][p][0];
                    u += sm.part[b][p][1];
                }
                const float av = (act == 1) ? fmaxf(g, 0.f) * u : g / (1.f + expf(-g)) * u;
                down_any(tier_of(j), ring + offs[b], d, av, y);
            }
        }
        __syncthreads();  // the batch's records are consumed; part[] reusable
        if (threadIdx.x == 0) {
            for (int b = 0; b < nb; b++) used -= sm.span[(j0 + b) % kNSlot];
            fence_proxy_async();
            issue_more(j0 + nb);
        }
        j0 += nb;
    }
    float *out = partial + (int64_t)blockIdx.x * d + 8 * threadIdx.x;
    reinterpret_cast<float4 *>(out)[0] = make_float4(y[0], y[1], y[2], y[3]);
    reinterpret_cast<float4 *>(out)[1] = make_float4(y[4], y[5], y[6], y[7]);
}

// ---- list-driven FFN (API path: m2c_sparse_ffn_forward, LRU hits / misses) --------------
__global__ void __launch_bounds__(1024, 1)
    k_ffn(FfnArgs a, int d, int act, const __half *__restrict__ x, const int32_t *__restrict__ items,
          const int32_t *__restrict__ counts, float *__restrict__ partial) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    uint8_t *ring = smem;
    uint4 *xs = reinterpret_cast<uint4 *>(smem + kRingList);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kNSlot; i++) mbar_init(&sm.bars[i], 1);
        fence_mbar_init();
    }
    griddep_launch();
    griddep_wait();
    if (threadIdx.x == 0) {
        int r[6];
        cta_ranges(a, counts[0], counts[1], counts[2], blockIdx.x, gridDim.x, r);
        for (int i = 0; i < 6; i++) sm.rng[i] = r[i];
    }
    __syncthreads();
    const int a0 = sm.rng[0], a1 = sm.rng[2], a2 = sm.rng[4];
    const int c1 = sm.rng[1] - a0, c2 = c1 + sm.rng[3] - a1, n_items = c2 + sm.rng[5] - a2;
    auto src = [&](int j) -> const uint8_t * {
        if (j < c1) return a.pool[0] + (int64_t)items[a.seg[0] + a0 + j] * a.nb[0];
        if (j < c2) return a.pool[1] + (int64_t)items[a.seg[1] + a1 + (j - c1)] * a.nb[1];
        return a.pool[2] + (int64_t)items[a.seg[2] + a2 + (j - c2)] * a.nb[2];
    };
    ffn_loop<kRingList>(a, d, act, x, n_items, c1, c2, src, ring, xs, sm, partial);
}

// ---- decode path: select (tier lists from scores + histogram) fused with the FFN ----------
__global__ void __launch_bounds__(1024, 1)
    k_ffn_sel(FfnArgs a, SelArgs s, int d, int act, const __half *__restrict__ x,
              float *__restrict__ partial) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    uint8_t *ring = smem;
    uint4 *xs = reinterpret_cast<uint4 *>(smem + kRingSel);           // [d/8], 16 KB reserved
    int *loc = reinterpret_cast<int *>(smem + kRingSel + 16384);     // [kMaxLocal]
    // the select scratch lives in the ring (unused until the records are requested)
    int *hist = reinterpret_cast<int *>(smem);                       // [4096]
    int *sub = hist + kHistBins;                                     // [3][2^sh]
    const int T = blockDim.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int n0 = s.k16, n1 = s.k8, n2 = s.k - s.k16 - s.k8;
    if (tid == 0) {
        for (int i = 0; i < kNSlot; i++) mbar_init(&sm.bars[i], 1);
        fence_mbar_init();
        int r[6];
        cta_ranges(a, n0, n1, n2, blockIdx.x, gridDim.x, r);
        for (int i = 0; i < 6; i++) sm.rng[i] = r[i];
    }
    __syncthreads();
    const int a0 = sm.rng[0], a1 = sm.rng[2], a2 = sm.rng[4];
    const int c1 = sm.rng[1] - a0, c2 = c1 + sm.rng[3] - a1, n_items = c2 + sm.rng[5] - a2;
    // speculative L2 prefetch of the records the previous token selected (hint only)
    if (warp == 1 && s.prev_ids) {
        for (int j = lane; j < n_items; j += 32) {
            int t, id;
            if (j < c1) { t = 0; id = s.prev_ids[a0 + j]; }
            else if (j < c2) { t = 1; id = s.prev_ids[n0 + a1 + (j - c1)]; }
            else { t = 2; id = s.prev_ids[n0 + n1 + a2 + (j - c2)]; }
            if (id >= 0 && id < s.F_r) {
                const uint8_t *p = a.pool[t] + (int64_t)id * a.nb[t];
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(a.nb[t]) : "memory");
            }
        }
    }
    griddep_launch();
    griddep_wait();

    // ---- 1. histogram -> bin holding the target-th largest, for the three targets ----
    const int tg[3] = {s.k16, s.k16 + s.k8, s.k};
    const int BPT = (kHistBins + T - 1) / T;
    int lsum = 0;
    for (int i = 0; i < BPT; i++) {  // descending bins: thread t covers [4095 - t*BPT - i]
        const int b = kHistBins - 1 - (tid * BPT + i);
        const int v = b >= 0 ? s.hist[b] : 0;
        if (b >= 0) hist[b] = v;
        lsum += v;
    }
    {
        int vv[3] = {lsum, 0, 0}, ex[3], tot[3];
        block_scan3(vv, ex, tot, sm.scan);
        int cum = ex[0];
        for (int i = 0; i < BPT; i++) {
            const int b = kHistBins - 1 - (tid * BPT + i);
            if (b < 0) break;
            const int v = hist[b];
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (tg[t] > 0 && cum < tg[t] && cum + v >= tg[t]) {
                    sm.selv[t] = b;          // bin
                    sm.selv[3 + t] = cum;    // elements above the bin
                }
            cum += v;
        }
    }
    const int nsub = 1 << s.sh;
    for (int i = tid; i < 3 * nsub; i += T) sub[i] = 0;
    __syncthreads();
    int bin[3], need[3];
#pragma unroll
    for (int t = 0; t < 3; t++) {
        bin[t] = tg[t] > 0 ? sm.selv[t] : -1;
        need[t] = tg[t] > 0 ? tg[t] - sm.selv[3 + t] : 0;
    }
    // ---- 2. second level: exact values inside the chosen bins ----
    for (int n = tid; n < s.F_r; n += T) {
        const int v = s.scores[n] + s.smax;
        const int b = v >> s.sh;
#pragma unroll
        for (int t = 0; t < 3; t++)
            if (b == bin[t]) atomicAdd(&sub[t * nsub + (v & (nsub - 1))], 1);
    }
    __syncthreads();
    if (warp < 3 && tg[warp] > 0) {  // warp t scans sub[t] from the top for need[t]
        const int t = warp;
        const int per = nsub / 32;
        int loc_sum = 0;
        for (int i = 0; i < per; i++) loc_sum += sub[t * nsub + nsub - 1 - (lane * per + i)];
        int inc = loc_sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y2 = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y2;
        }
        const int excl = inc - loc_sum;
        if (excl < need[t] && inc >= need[t]) {
            int cum = excl;
            for (int i = 0; i < per; i++) {
                const int c = nsub - 1 - (lane * per + i);
                const int v = sub[t * nsub + c];
                if (cum + v >= need[t]) {
                    sm.selv[6 + t] = (bin[t] << s.sh) | c;  // exact biased value V_t
                    sm.selv[9 + t] = need[t] - cum;         // how many equal to V_t are in
                    break;
                }
                cum += v;
            }
        }
    }
    __syncthreads();
    int V[3], R[3];
#pragma unroll
    for (int t = 0; t < 3; t++) {
        V[t] = tg[t] > 0 ? sm.selv[6 + t] : 0x7fffffff;
        R[t] = tg[t] > 0 ? sm.selv[9 + t] : 0;
    }
    // ---- 3. classify in id order, compact; keep this CTA's records, CTA 0 writes the lists ----
    const int CH = (s.F_r + T - 1) / T;
    const int i0 = min(s.F_r, tid * CH), i1 = min(s.F_r, i0 + CH);
    int eqv[3] = {0, 0, 0}, eqx[3], tot[3];
    for (int n = i0; n < i1; n++) {
        const int v = s.scores[n] + s.smax;
#pragma unroll
        for (int t = 0; t < 3; t++) eqv[t] += (v == V[t]);
    }
    block_scan3(eqv, eqx, tot, sm.scan);
    int cnt[3] = {0, 0, 0};
    for (int n = i0; n < i1; n++) {
        const int v = s.scores[n] + s.smax;
        int tr = -1;
#pragma unroll
        for (int t = 2; t >= 0; t--) {
            bool in = v > V[t];
            if (v == V[t]) in = (eqx[t]++ < R[t]);
            if (in) tr = t;
        }
        if (tr >= 0) cnt[tr]++;
    }
    int pos[3], tot2[3];
    block_scan3(cnt, pos, tot2, sm.scan);
    // re-walk (recomputing the equal-key ranks) to emit positions
    eqx[0] = eqx[0] - eqv[0];
    eqx[1] = eqx[1] - eqv[1];
    eqx[2] = eqx[2] - eqv[2];
    const int segs[3] = {0, n0, n0 + n1};
    const int lo_t[3] = {a0, a1, a2}, hi_t[3] = {a0 + c1, a1 + (c2 - c1), a2 + (n_items - c2)};
    const int lb_t[3] = {0, c1, c2};
    for (int n = i0; n < i1; n++) {
        const int v = s.scores[n] + s.smax;
        int tr = -1;
#pragma unroll
        for (int t = 2; t >= 0; t--) {
            bool in = v > V[t];
            if (v == V[t]) in = (eqx[t]++ < R[t]);
            if (in) tr = t;
        }
        if (tr >= 0) {
            int p = 0, lo = 0, hi = 0, lb = 0, sg = 0;
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (t == tr) {
                    p = pos[t]++;
                    lo = lo_t[t];
                    hi = hi_t[t];
                    lb = lb_t[t];
                    sg = segs[t];
                }
            if (p >= lo && p < hi) loc[lb + p - lo] = n;
            if (blockIdx.x == 0 && s.out_ids) s.out_ids[sg + p] = n;
        }
    }
    __syncthreads();
    auto src = [&](int j) -> const uint8_t * {
        const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
        return a.pool[t] + (int64_t)loc[j] * a.nb[t];
    };
    ffn_loop<kRingSel>(a, d, act, x, n_items, c1, c2, src, ring, xs, sm, partial);
}

}  // namespace

static size_t sel_smem(int sh) {
    (void)sh;  // hist + 3 sub-histograms (<= 64 KB) live inside the ring
    return (size_t)kRingSel + 16384 + 4 * (size_t)kMaxLocal;
}

cudaError_t init_ffn_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingList + 16384);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_ffn_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem(12));
    return e;
}

// balancing weight of one record: bytes + lambda * 3d weights (lambda = 0.5 B per weight)
static void fill_args(m2c_ctx *c, const LayerState &L, const m2c_tier_plan &p, FfnArgs &a) {
    const int d = c->desc.d_model;
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8};
    for (int t = 0; t < 3; t++) {
        a.pool[t] = L.pool[t];
        a.nb[t] = (int)c->nb[t];
        a.seg[t] = seg[t];
        a.wt[t] = (int)((c->nb[t] + 3 * (int64_t)d / 2) / 16);
    }
}

cudaError_t launch_ffn(m2c_ctx *c, const LayerState &L, const __half *x, const int32_t *items,
                       const int32_t *counts, const m2c_tier_plan &p, float *partial,
                       cudaStream_t st) {
    const int d = c->desc.d_model;
    FfnArgs a;
    fill_args(c, L, p, a);
    cudaError_t e = launch_k(k_ffn, dim3(c->G), dim3(d / 8), (size_t)kRingList + 2 * (size_t)d, st, a, d,
                             c->desc.act, x, items, counts, partial);
    c->launch_counter++;
    return e;
}

bool ffn_sel_supported(m2c_ctx *c, const m2c_tier_plan &p) {
    // every CTA's share must fit the local item list; sh <= 12
    FfnArgs a;
    LayerState dummy;
    fill_args(c, dummy, p, a);
    const long long W = (long long)p.k_fp16 * a.wt[0] + (long long)p.k_int8 * a.wt[1] + (long long)p.k_int4 * a.wt[2];
    const long long per = W / c->G + 1;
    const int wmin = a.wt[2] < a.wt[1] ? (a.wt[2] < a.wt[0] ? a.wt[2] : a.wt[0]) : (a.wt[1] < a.wt[0] ? a.wt[1] : a.wt[0]);
    return per / wmin + 3 <= kMaxLocal && c->sel_sh <= 12;
}

cudaError_t launch_ffn_sel(m2c_ctx *c, const LayerState &L, const __half *x, const int32_t *scores,
                           const int32_t *hist, int32_t *out_ids, const int32_t *prev_ids,
                           const m2c_tier_plan &p, float *partial, cudaStream_t st) {
    const int d = c->desc.d_model;
    FfnArgs a;
    fill_args(c, L, p, a);
    SelArgs s;
    s.scores = scores;
    s.hist = hist;
    s.out_ids = out_ids;
    s.prev_ids = prev_ids;
    s.F_r = c->F_r;
    s.k = p.k;
    s.k16 = p.k_fp16;
    s.k8 = p.k_int8;
    s.smax = c->sel_smax;
    s.sh = c->sel_sh;
    cudaError_t e = launch_k(k_ffn_sel, dim3(c->G), dim3(d / 8), sel_smem(c->sel_sh), st, a, s, d,
                             c->desc.act, x, partial);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

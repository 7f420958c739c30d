// ffn_dev.cuh -- device code of the fused dequant-GEMV FFN (a6), shared by k_ffn (API /
// LRU path) and k_decode (persistent decode kernel).
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
//    SASS UBLKCP), one mbarrier per record, issued by one thread as ring space frees; the
//    issuing thread publishes each record's ring offset, and precomputes the batches.
//  * Batches of up to 16 records: gate/up dot products are warp-local (one warp, or up to
//    four warps splitting d, per record; warp-shuffle reductions only), then the
//    down-projection where thread t owns elements [8t, 8t+8) of y in registers.
//  * Dequant in registers, ~2 instructions per weight: codes become the fp16 value 1024 + q
//    (or 1024 + 16q for odd INT4 nibbles) by PRMT/LOP3 (magic-exponent trick); HFMA2 removes
//    the offset and zero point exactly; fma.rn.f32.f16 (SASS FHFMA) multiplies exact fp16
//    (q - z) by fp16 x with an exact product and fp32 accumulation.  Per 128-group
//    s * sum (q - z) x (R5).
//  * The per-CTA partial y goes to a [G][d] fp32 buffer reduced in a fixed order by k_reduce.
#pragma once
#include <type_traits>
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kNBMax = 16;   // records per batch
#ifndef M2C_FFN_WS
#define M2C_FFN_WS 0         // warp-specialised fast path (gate/up warps | down warps): measured
                             // slower at S7 (gate/up on half the warps is the longer chain)
#endif
#ifndef M2C_FFN_STREAM_PREFETCH
#define M2C_FFN_STREAM_PREFETCH 0  // streaming path: L2 prefetch of the whole share up front (measured slower at S70H)
#endif
#ifndef M2C_FFN_STREAM_DIV
#define M2C_FFN_STREAM_DIV 0  // streaming path: batches of <= kRing / DIV bytes (0: ring - largest record)
#endif
#ifndef M2C_FFN_STREAM_PIPE
#define M2C_FFN_STREAM_PIPE 0  // streaming path: 1 = records released one by one as consumed (bit-identical, measured slower)
#endif
#ifndef M2C_FFN_STREAM_AHEAD
#define M2C_FFN_STREAM_AHEAD 0  // streaming path: L2 prefetch distance in records (0: off)
#endif
#ifndef M2C_FFN_FB_MUL
#define M2C_FFN_FB_MUL 4     // fast-path batch = M2C_FFN_FB_MUL x (warps / quarter-units per record); 1 measured slower (tools/exp_fb.sh)
#endif
#ifndef M2C_FFN_PBIG
#define M2C_FFN_PBIG 4       // max gate/up parts per record (8: d = 5120 / 8192 in 128-chunk parts -- measured neutral)
#endif
constexpr int kPMax = M2C_FFN_PBIG > 4 ? M2C_FFN_PBIG : 4;
// gate/up units per record: d / P elements per warp
// (128-chunk parts when d / 1024 <= kPMax: the 4-independent-chain path of gu_chunks)
__device__ __forceinline__ int ffn_parts(int nchunk) {
    if (nchunk % 128 == 0 && nchunk / 128 <= M2C_FFN_PBIG && nchunk >= 512) return nchunk / 128;
    return nchunk >= 512 ? 4 : 1;
}
constexpr int kNSlot = 32;   // mbarriers (>= records in flight)
constexpr int kRing = 192 * 1024;
constexpr int kMaxLocal = 1024;  // records one CTA may own
constexpr int kXsBytes = 16384;  // x (fp16, d <= 8192)
// dynamic smem: ring | xs | loc[kMaxLocal] | dsc[kMaxLocal] | bst[kMaxLocal + 1]
constexpr size_t kSmemBytes = (size_t)kRing + kXsBytes + 4 * (3 * kMaxLocal + 4);

struct FfnArgs {
    const uint8_t *pool[3];
    int nb[3];     // record bytes per tier
    int seg[3];    // tier segment offsets in the item lists
    int wt[3];     // balancing weight per record (bytes + lambda * 3d), in 16-B units
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
// (one 8-element chunk c into the accumulators ag, au)
template <int TIER>
__device__ __forceinline__ void gu_one(const uint8_t *rec, const uint4 *xs, int d, int c, float &ag, float &au);

template <int TIER>
__device__ __forceinline__ void gu_chunks(const uint8_t *rec, const uint4 *xs, int d, int c0, int c1,
                                          float &pg, float &pu) {
    const int lane = threadIdx.x & 31;
    if (c1 - c0 == 128) {  // the common quarter of d = 4096: 4 chunks per lane, independent chains
        float g0 = 0.f, u0 = 0.f, g1 = 0.f, u1 = 0.f, g2 = 0.f, u2 = 0.f, g3 = 0.f, u3 = 0.f;
        gu_one<TIER>(rec, xs, d, c0 + lane, g0, u0);
        gu_one<TIER>(rec, xs, d, c0 + lane + 32, g1, u1);
        gu_one<TIER>(rec, xs, d, c0 + lane + 64, g2, u2);
        gu_one<TIER>(rec, xs, d, c0 + lane + 96, g3, u3);
        pg = (g0 + g1) + (g2 + g3);
        pu = (u0 + u1) + (u2 + u3);
        return;
    }
    float ag = 0.f, au = 0.f;
    for (int c = c0 + lane; c < c1; c += 32) gu_one<TIER>(rec, xs, d, c, ag, au);
    pg = ag;
    pu = au;
}

template <int TIER>
__device__ __forceinline__ void gu_one(const uint8_t *rec, const uint4 *xs, int d, int c, float &ag, float &au) {
    const int G = d >> 7;
    {
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

// down-projection of batch records [ja, jb) of one tier (j0: the batch's first record)
template <int TIER>
__device__ __forceinline__ void down_seg(const uint8_t *ring, const int *dsc, const float *a_sm, int j0,
                                         int ja, int jb, int d, float (&y)[8]) {
    int j = ja;
    for (; j + 1 < jb; j += 2) {
        const int d0 = dsc[j], d1 = dsc[j + 1];
        const float a0 = a_sm[j - j0], a1 = a_sm[j + 1 - j0];
        down_t<TIER>(ring + (d0 & 0xffffff), d, a0, y);
        down_t<TIER>(ring + (d1 & 0xffffff), d, a1, y);
    }
    if (j < jb) down_t<TIER>(ring + (dsc[j] & 0xffffff), d, a_sm[j - j0], y);
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
    uint64_t abar[kNSlot];   // warp-specialised path: record j's activation a_j is ready
    int acnt[kNSlot];        // quarter-units of record j done
    int cons[kNSlot];        // streaming pipeline: warps done with record j's down-projection
    unsigned aflag[kNSlot];  // streaming pipeline: tag (jb + j + 1) once a_sm[slot] holds a_j
    int issued;              // streaming pipeline: records issued so far (thread 0 publishes)
    float apart[kNSlot][kPMax][2];
    int span[kNSlot];
    float part[kNBMax][kPMax][2];
    float a_sm[kNSlot];
    int cb[kPMax + 1][kPMax + 1];  // chunk bounds: cb[P][p] = nchunk * p / P
    int rng[8];          // CTA ranges (6)
    int nbatch;
    int scan[96];
    int selv[16];
};

__device__ __forceinline__ void ffn_init_bars(FfnShared &sm) {  // thread 0, before any use
    for (int i = 0; i < kNSlot; i++) {
        sm.aflag[i] = 0xffffffffu;
        mbar_init(&sm.bars[i], 1);
        mbar_init(&sm.abar[i], 1);
    }
    fence_mbar_init();
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// y[0..8) += a * deq(down column)[8 c8 .. 8 c8 + 8) (down_t for an explicit chunk of 8)
template <int TIER>
__device__ __forceinline__ void down_c(const uint8_t *rec, int d, float a, int c8, float *y) {
    if (TIER == 0) {
        const uint4 v = *reinterpret_cast<const uint4 *>(rec + 4 * d + 16 * c8);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            y[2 * i] = fmaf(a, h2f_lo(w[i]), y[2 * i]);
            y[2 * i + 1] = fmaf(a, h2f_hi(w[i]), y[2 * i + 1]);
        }
    } else {
        const int G = d >> 7, grp = c8 >> 4;
        const uint8_t *scales = rec + (TIER == 1 ? 3 * d : 3 * (d >> 1));
        const uint32_t z = (scales + 6 * G)[2 * G + grp];
        const float as = a * half_bits_f(*reinterpret_cast<const uint16_t *>(scales + 2 * (2 * G + grp)));
        uint32_t p[4];
        if (TIER == 1) {
            const uint2 v = *reinterpret_cast<const uint2 *>(rec + 2 * d + 8 * c8);
            deq8(v.x, v.y, zz2(z), p);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                y[2 * i] = fmaf(as, h2f_lo(p[i]), y[2 * i]);
                y[2 * i + 1] = fmaf(as, h2f_hi(p[i]), y[2 * i + 1]);
            }
        } else {
            const uint32_t w = *reinterpret_cast<const uint32_t *>(rec + d + 4 * c8);
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

// table: chunk bounds per split into P parts (constant for a launch)
__device__ __forceinline__ void ffn_tables(FfnShared &sm, int d) {
    const int nchunk = d / 8;
    if (threadIdx.x < (kPMax + 1) * (kPMax + 1)) {
        const int P = threadIdx.x / (kPMax + 1), p = threadIdx.x % (kPMax + 1);
        sm.cb[P][p] = P ? nchunk * p / P : 0;
    }
}

// The FFN main loop over this CTA's n_items records; item j -> global record pointer src(j).
// jb: mbarrier uses so far in this CTA (item j uses barrier (jb + j) % kNSlot in phase
// ((jb + j) / kNSlot) & 1), so a persistent kernel can run the loop once per layer.
// x == nullptr: xs already holds x.
template <class SrcFn>
__device__ __forceinline__ void ffn_loop(const FfnArgs &a, int d, int act, const __half *x, int n_items,
                                         int c1, int c2, SrcFn src, uint8_t *ring, uint4 *xs,
                                         int *dsc, int *bst, FfnShared &sm, float *partial,
                                         unsigned jb = 0, bool build_tables = true,
                                         unsigned long long *stamps = nullptr) {
    const int nwarp = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunk = d / 8;
    if (build_tables) ffn_tables(sm, d);
    // fast path: every record fits the ring at once -> warp 0 issues them in parallel (lane j:
    // record j, offsets by a warp prefix sum), batches of kNBMax
    const int total_bytes = c1 * a.nb[0] + (c2 - c1) * a.nb[1] + (n_items - c2) * a.nb[2];
    const bool fast = n_items <= kNSlot && total_bytes <= kRing;
    const uint64_t pol = policy_evict_first();
    if (fast) {
        if (threadIdx.x < 32) {
            const int j = threadIdx.x;
            const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
            const int sz = j < n_items ? a.nb[t] : 0;
            int inc = sz;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (j >= o) inc += y;
            }
            if (j < n_items) {
                const int off = inc - sz;
                dsc[j] = off | (t << 24);
                uint64_t *bar = &sm.bars[(jb + j) % kNSlot];
                // no proxy fence: callers order earlier generic ring writes (k_decode fences
                // before its FFN phase; k_ffn's ring has none)
                mbar_expect_tx(bar, (uint32_t)sz);
                bulk_g2s(ring + off, src(j), (uint32_t)sz, bar, pol);
            }
            // batches of one record per warp (P quarter-units each): the down-projection of a
            // batch overlaps the arrival of the next batch's records
            const int FB = max(1, min(kNBMax, (nwarp / ffn_parts(nchunk)) * M2C_FFN_FB_MUL));
            const int nbt = (n_items + FB - 1) / FB;
            if (j == 0) sm.nbatch = nbt;
            if (j <= nbt) bst[j] = min(j * FB, n_items);
        }
    } else if (threadIdx.x == 0) {
        // thread 0: batches (consecutive records that fit the ring together, with wrap slack)
        const int nbA = a.nb[0], nbB = a.nb[1], nbC = a.nb[2];
        const int mx = nbA > nbB ? (nbA > nbC ? nbA : nbC) : (nbB > nbC ? nbB : nbC);
        int nbt = 0;
        for (int j0 = 0; j0 < n_items;) {
            int nb = 0, bytes = 0;
            while (nb < kNBMax && j0 + nb < n_items) {
                const int j = j0 + nb;
                const int sz = j < c1 ? nbA : (j < c2 ? nbB : nbC);
#if M2C_FFN_STREAM_DIV
                // smaller batches: the next batch's copies land while this one computes
                if (nb > 0 && bytes + sz > kRing / M2C_FFN_STREAM_DIV) break;
#else
                if (nb > 0 && bytes + sz + mx > kRing) break;
#endif
                bytes += sz;
                nb++;
            }
            bst[nbt++] = j0;
            j0 += nb;
        }
        bst[nbt] = n_items;
        sm.nbatch = nbt;
    }
    // producer state (thread 0): bump allocation in the byte ring; publishes dsc[j]
    int issued = fast ? n_items : 0, pos_issue = 0, used = 0;
    auto issue_more = [&](int consumed) {
        while (issued < n_items && issued - consumed < kNSlot) {
            const int j = issued;
            const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
            const int sz = t == 0 ? a.nb[0] : (t == 1 ? a.nb[1] : a.nb[2]);
            const bool wrap = pos_issue + sz > kRing;  // (pos_issue == kRing wraps with no waste)
            const int waste = wrap ? kRing - pos_issue : 0;
            if (used + waste + sz > kRing) break;
            const int off = wrap ? 0 : pos_issue;
            sm.span[(jb + j) % kNSlot] = waste + sz;
            used += waste + sz;
            pos_issue = off + sz;
            dsc[j] = off | (t << 24);
            uint64_t *bar = &sm.bars[(jb + j) % kNSlot];
            mbar_expect_tx(bar, (uint32_t)sz);  // release: dsc[j] is visible to its waiters
            bulk_g2s(ring + off, src(j), (uint32_t)sz, bar, pol);
#if M2C_FFN_STREAM_AHEAD
            // the ring bounds the bytes in flight: pull the record M2C_FFN_STREAM_AHEAD places
            // later into L2 now (in TMA order after this copy), so its copy will hit L2
            if (j + M2C_FFN_STREAM_AHEAD < n_items) {
                const int j2 = j + M2C_FFN_STREAM_AHEAD;
                const int t2 = j2 < c1 ? 0 : (j2 < c2 ? 1 : 2);
                prefetch_l2(src(j2), (uint32_t)a.nb[t2]);
            }
#endif
            issued++;
        }
#if M2C_FFN_STREAM_PIPE
        *reinterpret_cast<volatile int *>(&sm.issued) = issued;
#endif
    };
#if M2C_FFN_STREAM_PIPE
    if (!fast && threadIdx.x < kNSlot) {
        sm.cons[threadIdx.x] = 0;
        sm.acnt[threadIdx.x] = 0;
        if (threadIdx.x == 0) sm.issued = 0;
    }
#endif
    // x -> smem as fp16 (read by the warp-local dot products)
    if (x)
        for (int c = threadIdx.x; c < nchunk; c += blockDim.x) xs[c] = reinterpret_cast<const uint4 *>(x)[c];
    __syncthreads();
    if (stamps && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamps[0]));
    // streaming path: the first copies are issued after the barrier (a bulk-copy issue can stall
    // its thread while the TMA unit is busy; the other warps are already waiting on the records'
    // mbarriers, and each record's offset is published by its expect_tx arrival)
    if (threadIdx.x == 0 && !fast) {
        fence_proxy_async();
        issue_more(0);
    }
#if M2C_FFN_STREAM_PREFETCH
    // streaming path: the ring (192 KB) bounds the bytes in flight, so the share's later
    // records are pulled into L2 now by warp 1 (per-line prefetches, no smem), and the ring's
    // copies then hit L2
    if (!fast && warp == 1) {
        for (int j = 0; j < n_items; j++) {
            const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
            const char *g = reinterpret_cast<const char *>(src(j));
            for (int o = 128 * lane; o < a.nb[t]; o += 128 * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(g + o));
        }
    }
#endif

#if M2C_FFN_STREAM_PIPE
    if (!fast) {
        // Streaming pipeline (the share exceeds the ring): ring space is released record by
        // record, in order, as soon as every warp has done its down-projection of it, so the
        // copies of later records stream in continuously instead of batch by batch.  Each warp
        // computes its gate/up units (record j, part pp dealt round-robin) of every ISSUED
        // record as the copies land; the last part of a record combines the parts in a fixed
        // order and publishes a_j (tag aflag); every warp then accumulates the down-projection
        // of its 8 y elements per thread record by record in ascending j.  Per element the
        // operations and their order are the batched path's (bit-identical).  Thread 0 is also
        // the producer: whenever it would wait it frees consumed records and issues more, so no
        // wait can block the copies it depends on.
        const int P = ffn_parts(nchunk);
        int freed = 0;
        auto produce = [&]() {  // thread 0 only
            bool any = false;
            while (freed < issued &&
                   *reinterpret_cast<volatile int *>(&sm.cons[(jb + freed) % kNSlot]) == nwarp) {
                sm.cons[(jb + freed) % kNSlot] = 0;
                used -= sm.span[(jb + freed) % kNSlot];
                freed++;
                any = true;
            }
            if (any) {
                fence_proxy_async();  // the consumers' generic ring reads precede the new copies
                issue_more(freed);
            }
        };
        const bool prod = threadIdx.x == 0;
        auto wait_bar = [&](uint64_t *bar, uint32_t par) {
            if (prod) {
                while (!mbar_test(bar, par)) produce();
            } else {
                mbar_wait(bar, par);
            }
        };
        float y[8];
#pragma unroll
        for (int i = 0; i < 8; i++) y[i] = 0.f;
        int u = warp;  // this warp's next gate/up unit: record u / P, part u % P
        for (int j = 0; j < n_items; j++) {
            // gate/up units of every issued record (and at least of record j)
            for (;;) {
                if (u >= n_items * P) break;
                const int jj = u / P, pp = u - jj * P;
                if (jj > j) {  // (one read for the whole warp: the decision must be uniform)
                    const int is = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile int *>(&sm.issued), 0);
                    if (jj >= is) break;
                } else {
                    while (jj >= *reinterpret_cast<volatile int *>(&sm.issued))
                        if (prod) produce();
                }
                const unsigned sl = (jb + jj) % kNSlot;
                wait_bar(&sm.bars[sl], ((jb + jj) / kNSlot) & 1);
                const int ds = dsc[jj];
                float pg, pu;
                gu_any(ds >> 24, ring + (ds & 0xffffff), xs, d, sm.cb[P][pp], sm.cb[P][pp + 1], pg, pu);
                pg = warp_sum_f(pg);
                pu = warp_sum_f(pu);
                if (lane == 0) {
                    sm.apart[sl][pp][0] = pg;
                    sm.apart[sl][pp][1] = pu;
                    __threadfence_block();
                    if (atomicAdd(&sm.acnt[sl], 1) == P - 1) {  // last part: combine, publish
                        __threadfence_block();
                        float g = 0.f, uu = 0.f;
                        for (int q = 0; q < P; q++) {
                            g += sm.apart[sl][q][0];
                            uu += sm.apart[sl][q][1];
                        }
                        sm.acnt[sl] = 0;
                        sm.a_sm[sl] = (act == 1) ? fmaxf(g, 0.f) * uu : g / (1.f + expf(-g)) * uu;
                        __threadfence_block();
                        *reinterpret_cast<volatile unsigned *>(&sm.aflag[sl]) = jb + (unsigned)jj + 1u;
                    }
                }
                __syncwarp();
                u += nwarp;
            }
            // down-projection of record j (ascending j: the batched path's order)
            const unsigned sl = (jb + j) % kNSlot, tag = jb + (unsigned)j + 1u;
            while (*reinterpret_cast<volatile unsigned *>(&sm.aflag[sl]) != tag)
                if (prod) produce();
            __threadfence_block();
            const int ds = dsc[j];
            const float aj = *reinterpret_cast<volatile float *>(&sm.a_sm[sl]);
            const int tier = ds >> 24;
            if (tier == 0) down_t<0>(ring + (ds & 0xffffff), d, aj, y);
            else if (tier == 1) down_t<1>(ring + (ds & 0xffffff), d, aj, y);
            else down_t<2>(ring + (ds & 0xffffff), d, aj, y);
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                atomicAdd(&sm.cons[sl], 1);
            }
            if (prod) produce();
        }
        if (stamps && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamps[1]));
        float *out = partial + (int64_t)blockIdx.x * d + 8 * threadIdx.x;
        reinterpret_cast<float4 *>(out)[0] = make_float4(y[0], y[1], y[2], y[3]);
        reinterpret_cast<float4 *>(out)[1] = make_float4(y[4], y[5], y[6], y[7]);
        __syncthreads();  // the ring's records are consumed
        return;
    }
#endif
    if (fast && M2C_FFN_WS == 2) {
        // Pipelined (all records in flight): every warp first computes its gate/up units in
        // record order as the copies land (the unit that completes record j combines its
        // quarters in a fixed order and arrives on abar[j]), then accumulates the
        // down-projection of its own 8 y elements per thread record by record, waiting only
        // for each a_j -- no block-wide barrier between the two, so the down-projection of
        // the early records overlaps the gate/up of the late ones.  Per element the
        // operations and their order are those of the batched path (bit-identical).
        const int P = ffn_parts(nchunk);
        if (threadIdx.x < kNSlot) sm.acnt[threadIdx.x] = 0;
        __syncthreads();
        for (int u = warp; u < n_items * P; u += nwarp) {
            const int j = u / P, pp = u - j * P;
            mbar_wait(&sm.bars[(jb + j) % kNSlot], (uint32_t)(((jb + j) / kNSlot) & 1));
            const int ds = dsc[j];
            float pg, pu;
            gu_any(ds >> 24, ring + (ds & 0xffffff), xs, d, sm.cb[P][pp], sm.cb[P][pp + 1], pg, pu);
            pg = warp_sum_f(pg);
            pu = warp_sum_f(pu);
            if (lane == 0) {
                if (P == 1) {
                    sm.a_sm[j] = (act == 1) ? fmaxf(pg, 0.f) * pu : pg / (1.f + expf(-pg)) * pu;
                    mbar_arrive(&sm.abar[(jb + j) % kNSlot]);
                } else {
                    sm.apart[j][pp][0] = pg;
                    sm.apart[j][pp][1] = pu;
                    __threadfence_block();
                    if (atomicAdd(&sm.acnt[j], 1) == P - 1) {  // last quarter: combine, publish
                        __threadfence_block();
                        float g = 0.f, uu = 0.f;
                        for (int q = 0; q < P; q++) {
                            g += sm.apart[j][q][0];
                            uu += sm.apart[j][q][1];
                        }
                        sm.a_sm[j] = (act == 1) ? fmaxf(g, 0.f) * uu : g / (1.f + expf(-g)) * uu;
                        mbar_arrive(&sm.abar[(jb + j) % kNSlot]);
                    }
                }
            }
        }
        if (stamps && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamps[1]));
        float y[8];
#pragma unroll
        for (int i = 0; i < 8; i++) y[i] = 0.f;
        // the batched path's order: tier segments, two records per step
        auto wait_a = [&](int j) { mbar_wait(&sm.abar[(jb + j) % kNSlot], (uint32_t)(((jb + j) / kNSlot) & 1)); };
        auto down_range = [&](auto tier_c, int ja, int jz) {
            constexpr int TIER = decltype(tier_c)::value;
            int j = ja;
            for (; j + 1 < jz; j += 2) {
                wait_a(j);
                wait_a(j + 1);
                const int d0 = dsc[j], d1 = dsc[j + 1];
                const float a0 = sm.a_sm[j], a1 = sm.a_sm[j + 1];
                down_t<TIER>(ring + (d0 & 0xffffff), d, a0, y);
                down_t<TIER>(ring + (d1 & 0xffffff), d, a1, y);
            }
            if (j < jz) {
                wait_a(j);
                down_t<TIER>(ring + (dsc[j] & 0xffffff), d, sm.a_sm[j], y);
            }
        };
        // (batches of the batched path: [bst[b], bst[b+1]); inside, tier segments)
        const int nbt = sm.nbatch;
        for (int bi = 0; bi < nbt; bi++) {
            const int j0 = bst[bi], je = bst[bi + 1];
            const int s1 = min(max(c1, j0), je), s2 = min(max(c2, j0), je);
            down_range(std::integral_constant<int, 0>(), j0, s1);
            down_range(std::integral_constant<int, 1>(), s1, s2);
            down_range(std::integral_constant<int, 2>(), s2, je);
        }
        float *out = partial + (int64_t)blockIdx.x * d + 8 * threadIdx.x;
        reinterpret_cast<float4 *>(out)[0] = make_float4(y[0], y[1], y[2], y[3]);
        reinterpret_cast<float4 *>(out)[1] = make_float4(y[4], y[5], y[6], y[7]);
        __syncthreads();  // the ring's records are consumed
        return;
    }
    if (fast && nwarp >= 2 && (nwarp & 1) == 0 && M2C_FFN_WS == 1) {
        // Warp-specialised (all records in flight): warps [0, NG) compute gate/up units in
        // record order as the copies land; the unit that completes record j combines its
        // quarters in a fixed order and arrives on abar[j]; warps [NG, nwarp) own 2 x 8 y
        // elements per thread and accumulate the down-projection record by record as each
        // a_j becomes ready -- the down-projection overlaps the arrival of later records.
        // Per element the operations and their order are those of the batched path.
        const int P = ffn_parts(nchunk);
        const int NG = nwarp / 2;
        if (threadIdx.x < kNSlot) sm.acnt[threadIdx.x] = 0;
        __syncthreads();
        if (warp < NG) {
            for (int u = warp; u < n_items * P; u += NG) {
                const int j = u / P, pp = u - j * P;
                mbar_wait(&sm.bars[(jb + j) % kNSlot], (uint32_t)(((jb + j) / kNSlot) & 1));
                const int ds = dsc[j];
                float pg, pu;
                gu_any(ds >> 24, ring + (ds & 0xffffff), xs, d, sm.cb[P][pp], sm.cb[P][pp + 1], pg, pu);
                pg = warp_sum_f(pg);
                pu = warp_sum_f(pu);
                if (lane == 0) {
                    sm.apart[j][pp][0] = pg;
                    sm.apart[j][pp][1] = pu;
                    __threadfence_block();
                    if (atomicAdd(&sm.acnt[j], 1) == P - 1) {  // last quarter: combine, publish
                        __threadfence_block();
                        float g = 0.f, uu = 0.f;
                        for (int q = 0; q < P; q++) {
                            g += sm.apart[j][q][0];
                            uu += sm.apart[j][q][1];
                        }
                        sm.a_sm[j] = (act == 1) ? fmaxf(g, 0.f) * uu : g / (1.f + expf(-g)) * uu;
                        mbar_arrive(&sm.abar[(jb + j) % kNSlot]);
                    }
                }
            }
            if (stamps && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamps[1]));
        } else {
            const int t2 = threadIdx.x - NG * 32;  // 0 .. (nwarp - NG) * 32
            const int c8a = 2 * t2, c8b = 2 * t2 + 1;
            float ya[8], yb[8];
#pragma unroll
            for (int i = 0; i < 8; i++) ya[i] = yb[i] = 0.f;
            for (int j = 0; j < n_items; j++) {
                mbar_wait(&sm.abar[(jb + j) % kNSlot], (uint32_t)(((jb + j) / kNSlot) & 1));
                const int ds = dsc[j];
                const uint8_t *rec = ring + (ds & 0xffffff);
                const float aj = sm.a_sm[j];
                const int tier = ds >> 24;
                if (tier == 0) {
                    down_c<0>(rec, d, aj, c8a, ya);
                    down_c<0>(rec, d, aj, c8b, yb);
                } else if (tier == 1) {
                    down_c<1>(rec, d, aj, c8a, ya);
                    down_c<1>(rec, d, aj, c8b, yb);
                } else {
                    down_c<2>(rec, d, aj, c8a, ya);
                    down_c<2>(rec, d, aj, c8b, yb);
                }
            }
            float *out = partial + (int64_t)blockIdx.x * d + 16 * t2;
            reinterpret_cast<float4 *>(out)[0] = make_float4(ya[0], ya[1], ya[2], ya[3]);
            reinterpret_cast<float4 *>(out)[1] = make_float4(ya[4], ya[5], ya[6], ya[7]);
            reinterpret_cast<float4 *>(out)[2] = make_float4(yb[0], yb[1], yb[2], yb[3]);
            reinterpret_cast<float4 *>(out)[3] = make_float4(yb[4], yb[5], yb[6], yb[7]);
        }
        __syncthreads();  // the ring's records are consumed
        return;
    }
    float y[8];
#pragma unroll
    for (int i = 0; i < 8; i++) y[i] = 0.f;
    const int nbt = sm.nbatch;
    const int P = ffn_parts(nchunk);
    for (int bi = 0; bi < nbt; bi++) {
        const int j0 = bst[bi], nb = bst[bi + 1] - j0;
        // gate/up: units (record b, quarter p) dealt round-robin to the warps (a warp may take
        // several); each unit ends in a warp-shuffle reduction, quarters combine in order
        for (int u = warp; u < nb * P; u += nwarp) {
            const int b = u / P, pp = u - b * P;
            const int j = j0 + b;
            mbar_wait(&sm.bars[(jb + j) % kNSlot], (uint32_t)(((jb + j) / kNSlot) & 1));
            const int ds = dsc[j];
            float pg, pu;
#ifdef M2C_EXP_SKIP_GU  // measurement build only (tools/): data arrival without the dot products
            pg = pu = 0.f;
            (void)ds;
#else
            gu_any(ds >> 24, ring + (ds & 0xffffff), xs, d, sm.cb[P][pp], sm.cb[P][pp + 1], pg, pu);
#endif
            pg = warp_sum_f(pg);
            pu = warp_sum_f(pu);
            if (lane == 0) {
                if (P == 1) {
                    sm.a_sm[b] = (act == 1) ? fmaxf(pg, 0.f) * pu : pg / (1.f + expf(-pg)) * pu;
                } else {
                    sm.part[b][pp][0] = pg;
                    sm.part[b][pp][1] = pu;
                }
            }
        }
        __syncthreads();
        if (P > 1) {  // combine the parts of each record, fixed order
            if (threadIdx.x < nb) {
                const int b = threadIdx.x;
                float g = 0.f, u = 0.f;
                for (int p = 0; p < P; p++) {
                    g += sm.part[b][p][0];
                    u += sm.part[b][p][1];
                }
                sm.a_sm[b] = (act == 1) ? fmaxf(g, 0.f) * u : g / (1.f + expf(-g)) * u;
            }
            __syncthreads();
        }
        if (stamps && threadIdx.x == 0 && bi == nbt - 1)
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamps[1]));
        {  // per tier segment of the batch, two records per step (independent loads in flight)
            const int je = j0 + nb;
            const int s1 = min(max(c1, j0), je), s2 = min(max(c2, j0), je);
            down_seg<0>(ring, dsc, sm.a_sm, j0, j0, s1, d, y);
            down_seg<1>(ring, dsc, sm.a_sm, j0, s1, s2, d, y);
            down_seg<2>(ring, dsc, sm.a_sm, j0, s2, je, d, y);
        }
        __syncthreads();  // the batch's records are consumed; a_sm/part reusable
        if (threadIdx.x == 0) {
            for (int b = 0; b < nb; b++) used -= sm.span[(jb + j0 + b) % kNSlot];
            fence_proxy_async();
            issue_more(j0 + nb);
        }
    }
    float *out = partial + (int64_t)blockIdx.x * d + 8 * threadIdx.x;
    reinterpret_cast<float4 *>(out)[0] = make_float4(y[0], y[1], y[2], y[3]);
    reinterpret_cast<float4 *>(out)[1] = make_float4(y[4], y[5], y[6], y[7]);
}

struct SmemPtrs {
    uint8_t *ring;
    uint4 *xs;
    int *loc, *dsc, *bst;
};
__device__ __forceinline__ SmemPtrs carve(uint8_t *smem) {
    SmemPtrs p;
    p.ring = smem;
    p.xs = reinterpret_cast<uint4 *>(smem + kRing);
    p.loc = reinterpret_cast<int *>(smem + kRing + kXsBytes);
    p.dsc = p.loc + kMaxLocal;
    p.bst = p.dsc + kMaxLocal;
    return p;
}

}  // namespace

// balancing weight of one record, in 16-B units: bytes + lambda * 3d weights.  lambda = 6 B per
// weight fits the per-CTA FFN times measured inside k_decode (profiles/: ~0.9 us of dequant +
// FMA per record at any precision plus ~12 ns per KB), i.e. the split is close to per-record.
#ifndef M2C_FFN_LAMBDA
#define M2C_FFN_LAMBDA 6
#endif
constexpr int kLambda = M2C_FFN_LAMBDA;
static inline int ffn_weight(int64_t nb, int d) { return (int)((nb + (int64_t)kLambda * 3 * d) / 16); }
static inline void fill_args(m2c_ctx *c, const LayerState &L, const m2c_tier_plan &p, FfnArgs &a) {
    const int d = c->desc.d_model;
    const int seg[3] = {0, p.k_fp16, p.k_fp16 + p.k_int8};
    for (int t = 0; t < 3; t++) {
        a.pool[t] = L.pool[t];
        a.nb[t] = (int)c->nb[t];
        a.seg[t] = seg[t];
        a.wt[t] = ffn_weight(c->nb[t], d);
    }
}

}  // namespace m2c

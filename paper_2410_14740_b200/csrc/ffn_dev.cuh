// ffn_dev.cuh -- device code of the fused dequant-GEMV FFN (a6), shared by k_ffn (API / LRU
// path) and k_decode (the persistent decode kernel's P4 phase).
//
// Paper: a neuron is a row of the first FFN matrices and the matching column of the next
// (P:58); only the active neurons are computed; the cache unit memory "can be
// directly used for inference computation, avoiding unnecessary copying from the cache to
// inference tensors"; low-bit neurons are dequantised for compute.  Decode is
// memory-bound: batch-1 GEMV at ~1 flop/byte, so CUDA cores, not tensor cores.
//
// B200 design (one persistent CTA per SM, T = d/8 threads):
//  * Work split: each CTA owns a contiguous share of the active records (tier order FP16,
//    INT8, INT4), balanced on bytes + lambda * weights (an INT4 record has 1/4 of the bytes
//    of an FP16 one but the same 3d weights to dequantise).
//  * Two phases per share.  G: the gate/up dot products, in units (record j, part p: 2 KB of
//    each row's codes, i.e. 1024 FP16 / 2048 INT8 / 4096 INT4 elements, gu_unit) dealt
//    round-robin to the compute warps, each ending in warp shuffles; the warp completing a
//    record's last part combines the parts in a fixed order into a_j = act(g_j) u_j.  D: the
//    down-projection, thread t owning y[8t, 8t+8) in registers, records in share order --
//    every element's sum has a fixed order (bit-reproducible).
//  * Data movement by the TMA engine (cp.async.bulk, SASS UBLKCP) into a 192 KB shared-memory
//    ring with full / empty mbarriers per entry (whole mode: every record at once;
//    streaming mode: a producer warp streams the gate/up rows (+ tail) FIFO, re-using each
//    entry as soon as its units arrive, and prefetches the down rows into L2 for phase D's
//    loads) -- see ffn_run.  (Measured alternatives -- LDG streaming with and without software
//    pipelining, speculative gate/up on the previous token's share, L2 prefetch of predicted
//    records, the down rows by TMA into the freed ring, split G/D warp groups -- were slower:
//    profiles/r02_ffn_variants.txt.)
//  * Dequant in registers, ~2 instructions per weight: codes become the fp16 value 1024 + q
//    (or 1024 + 16q for odd INT4 nibbles) by PRMT/LOP3 (magic-exponent trick); HSUB2 removes
//    the offset and zero point exactly; fma.rn.f32.f16 (SASS FHFMA) multiplies exact fp16
//    (q - z) by fp16 x with an exact product and fp32 accumulation.  Per 128-group
//    s * sum (q - z) x (R5).
//  * The per-CTA partial y goes to a [G][d] fp32 buffer reduced in a fixed order.
#pragma once
#include <type_traits>

#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kRing = 192 * 1024;
constexpr int kNS = 64;          // pipeline entries in flight (full / empty mbarrier pairs)
constexpr int kPMax = 8;         // gate/up parts per record (<= 8 for d <= 8192, gu_parts)
constexpr int kMaxLocal = 1024;  // records one CTA may own
constexpr int kXsBytes = 16384;  // x (fp16, d <= 8192)
// dynamic smem: ring | xs | loc[kMaxLocal] | a[kMaxLocal]
constexpr size_t kSmemBytes = (size_t)kRing + kXsBytes + 8 * (size_t)kMaxLocal;

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

// ---- gate/up units --------------------------------------------------------------------
// A "chunk" is 16 B of one row's codes: 8 (FP16), 16 (INT8) or 32 (INT4) elements, inside one
// 128-element quantisation group.  A unit (record, part p) covers chunks [128 p, 128 p + 128)
// of the gate row and of the up row: lane L takes chunks 128 p + L + 32 u, u < 4 (LDS.128 of
// consecutive 16 B across the lanes: conflict-free), one scale / zero-point per chunk and row,
// x read from its natural fp16 copy (2 / 4 blocks of 16 B per INT8 / INT4 chunk; permuted
// conflict-free copies of x measured slower: their 32 KB came out of the ring).  Round 1 used
// 8-element chunks for every tier: 4 / 8-B code loads and a scale per 8 INT elements -- ~3.75
// instructions per INT4 weight, the INT-heavy shares' P4 being issue-bound at S70H
// (profiles/r02_ffn_variants.txt).
__device__ __forceinline__ int row_bytes(int t, int d) { return t == 0 ? 2 * d : (t == 1 ? d : d / 2); }
__device__ __forceinline__ int gu_parts(int t, int d) { return (row_bytes(t, d) / 16 + 127) >> 7; }
__device__ __forceinline__ void fma16x2(float &acc, uint32_t a, uint32_t b) {  // acc += a.lo b.lo + a.hi b.hi
    hfma32(acc, a, b, 0, 0);
    hfma32(acc, a, b, 1, 1);
}
// INT4 word w (elements 0..7 in nibbles 0..7) against the x block xb (elements 0..7): deq4
// pairs (e0,e4), 16(e1,e5), (e2,e6), 16(e3,e7) (exact fp16 q - z); the 16x terms go to t16
__device__ __forceinline__ void int4_word(uint32_t w, uint32_t zz, uint32_t zz16, const uint4 &xb, float &t,
                                          float &t16) {
    uint32_t q[4];
    deq4(w, zz, zz16, q);
    hfma32(t, q[0], xb.x, 0, 0);
    hfma32(t, q[0], xb.z, 1, 0);
    hfma32(t16, q[1], xb.x, 0, 1);
    hfma32(t16, q[1], xb.z, 1, 1);
    hfma32(t, q[2], xb.y, 0, 0);
    hfma32(t, q[2], xb.w, 1, 0);
    hfma32(t16, q[3], xb.y, 0, 1);
    hfma32(t16, q[3], xb.w, 1, 1);
}
// gr / ur: the record's gate / up row in shared memory (row_bytes each); tail: its scale /
// zero tail (scales fp16[3G] | zeros u8[3G]).  (pg, pu): the part's dot products, warp-summed.
template <int T>
__device__ __forceinline__ void gu_unit(const uint8_t *gr, const uint8_t *ur, const uint8_t *tail, int d, int p,
                                        const uint4 *x16, float &pg, float &pu) {
    const int lane = threadIdx.x & 31;
    const int nch = row_bytes(T, d) >> 4, G = d >> 7;
    const int c0 = p << 7;
    float ag[4], au[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
        const int c = c0 + lane + 32 * u;
        const bool in = c < nch;
        const int cc = in ? c : 0;
        const uint4 gv = *reinterpret_cast<const uint4 *>(gr + 16 * cc);
        const uint4 uv = *reinterpret_cast<const uint4 *>(ur + 16 * cc);
        if (T == 0) {
            const uint4 xv = x16[cc];
            float g = 0.f, v = 0.f;
            fma16x2(g, gv.x, xv.x);
            fma16x2(g, gv.y, xv.y);
            fma16x2(g, gv.z, xv.z);
            fma16x2(g, gv.w, xv.w);
            fma16x2(v, uv.x, xv.x);
            fma16x2(v, uv.y, xv.y);
            fma16x2(v, uv.z, xv.z);
            fma16x2(v, uv.w, xv.w);
            ag[u] = in ? g : 0.f;
            au[u] = in ? v : 0.f;
        } else {
            const int grp = T == 1 ? cc >> 3 : cc >> 2;
            const uint16_t *s16 = reinterpret_cast<const uint16_t *>(tail);
            const uint8_t *z8 = tail + 6 * G;
            const float sg = half_bits_f(s16[grp]), su = half_bits_f(s16[G + grp]);
            const uint32_t zg = z8[grp], zu = z8[G + grp];
            float tg = 0.f, tu = 0.f;
            if (T == 1) {
                const uint4 xa = x16[2 * cc], xc = x16[2 * cc + 1];
                uint32_t qg[4], qu[4];
                const uint32_t zzg = zz2(zg), zzu = zz2(zu);
                deq8(gv.x, gv.y, zzg, qg);
                deq8(uv.x, uv.y, zzu, qu);
                fma16x2(tg, qg[0], xa.x);
                fma16x2(tg, qg[1], xa.y);
                fma16x2(tg, qg[2], xa.z);
                fma16x2(tg, qg[3], xa.w);
                fma16x2(tu, qu[0], xa.x);
                fma16x2(tu, qu[1], xa.y);
                fma16x2(tu, qu[2], xa.z);
                fma16x2(tu, qu[3], xa.w);
                deq8(gv.z, gv.w, zzg, qg);
                deq8(uv.z, uv.w, zzu, qu);
                fma16x2(tg, qg[0], xc.x);
                fma16x2(tg, qg[1], xc.y);
                fma16x2(tg, qg[2], xc.z);
                fma16x2(tg, qg[3], xc.w);
                fma16x2(tu, qu[0], xc.x);
                fma16x2(tu, qu[1], xc.y);
                fma16x2(tu, qu[2], xc.z);
                fma16x2(tu, qu[3], xc.w);
            } else {
                const uint4 *xb = x16 + 4 * cc;
                const uint32_t zzg = zz2(zg), zzg16 = zz2_16(zg), zzu = zz2(zu), zzu16 = zz2_16(zu);
                float tg16 = 0.f, tu16 = 0.f;
                const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w}, uw[4] = {uv.x, uv.y, uv.z, uv.w};
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint4 xk = xb[k];
                    int4_word(gw[k], zzg, zzg16, xk, tg, tg16);
                    int4_word(uw[k], zzu, zzu16, xk, tu, tu16);
                }
                tg = fmaf(tg16, 0.0625f, tg);
                tu = fmaf(tu16, 0.0625f, tu);
            }
            ag[u] = in ? sg * tg : 0.f;
            au[u] = in ? su * tu : 0.f;
        }
    }
    pg = warp_sum_f((ag[0] + ag[1]) + (ag[2] + ag[3]));
    pu = warp_sum_f((au[0] + au[1]) + (au[2] + au[3]));
}
__device__ __forceinline__ void gu_unit_any(int t, const uint8_t *gr, const uint8_t *ur, const uint8_t *tail, int d,
                                            int p, const uint4 *x16, float &pg, float &pu) {
    if (t == 0) gu_unit<0>(gr, ur, tail, d, p, x16, pg, pu);
    else if (t == 1) gu_unit<1>(gr, ur, tail, d, p, x16, pg, pu);
    else gu_unit<2>(gr, ur, tail, d, p, x16, pg, pu);
}

// ---- y[8t .. 8t+8) += a * deq(down column) from shared memory --------------------------
// e: the down data (whole record + 2D, or a streamed down entry); sc: its scale/zero tail
template <int TIER>
__device__ __forceinline__ void down_acc(const uint8_t *e, const uint8_t *sc, int d, float a, float (&y)[8]) {
    const int t = threadIdx.x;
    if (TIER == 0) {
        const uint4 v = *reinterpret_cast<const uint4 *>(e + 16 * t);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            y[2 * i] = fmaf(a, h2f_lo(w[i]), y[2 * i]);
            y[2 * i + 1] = fmaf(a, h2f_hi(w[i]), y[2 * i + 1]);
        }
    } else {
        const int G = d >> 7, grp = t >> 4;
        const float as = a * half_bits_f(*reinterpret_cast<const uint16_t *>(sc + 2 * (2 * G + grp)));
        const uint32_t z = sc[6 * G + 2 * G + grp];
        uint32_t p[4];
        if (TIER == 1) {
            const uint2 v = *reinterpret_cast<const uint2 *>(e + 8 * t);
            deq8(v.x, v.y, zz2(z), p);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                y[2 * i] = fmaf(as, h2f_lo(p[i]), y[2 * i]);
                y[2 * i + 1] = fmaf(as, h2f_hi(p[i]), y[2 * i + 1]);
            }
        } else {
            const uint32_t w = *reinterpret_cast<const uint32_t *>(e + 4 * t);
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

// ---- the same from global memory (whole-record layout), several records' loads in flight --
template <int TIER>
struct DownLd {
    uint4 v;
    float s;
    uint32_t z;
};
__device__ __forceinline__ uint4 ld_dn16(const void *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_dn8(const void *p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned ld_dn4(const void *p) {
    unsigned v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <int TIER>
__device__ __forceinline__ void down_ldg(const uint8_t *rec, int d, DownLd<TIER> &o) {
    const int t = threadIdx.x;
    if (TIER == 0) {
        o.v = ld_dn16(rec + 4 * d + 16 * t);
    } else {
        const int G = d >> 7, grp = t >> 4;
        const int D = TIER == 1 ? d : d / 2;
        const uint8_t *sc = rec + 3 * D;
        if (TIER == 1) {
            const uint2 w = ld_dn8(rec + 2 * d + 8 * t);
            o.v = make_uint4(w.x, w.y, 0, 0);
        } else {
            o.v = make_uint4(ld_dn4(rec + d + 4 * t), 0, 0, 0);
        }
        const unsigned short *sp = reinterpret_cast<const unsigned short *>(sc + 2 * (2 * G + grp));
        const unsigned char *zp = sc + 6 * G + 2 * G + grp;
        o.s = half_bits_f(__ldg(sp));
        o.z = __ldg(zp);
    }
}
template <int TIER>
__device__ __forceinline__ void down_fma(const DownLd<TIER> &o, float a, float (&y)[8]) {
    if (TIER == 0) {
        const uint32_t w[4] = {o.v.x, o.v.y, o.v.z, o.v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            y[2 * i] = fmaf(a, h2f_lo(w[i]), y[2 * i]);
            y[2 * i + 1] = fmaf(a, h2f_hi(w[i]), y[2 * i + 1]);
        }
    } else {
        const float as = a * o.s;
        uint32_t p[4];
        if (TIER == 1) {
            deq8(o.v.x, o.v.y, zz2(o.z), p);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                y[2 * i] = fmaf(as, h2f_lo(p[i]), y[2 * i]);
                y[2 * i + 1] = fmaf(as, h2f_hi(p[i]), y[2 * i + 1]);
            }
        } else {
            deq4(o.v.x, zz2(o.z), zz2_16(o.z), p);
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
// records [ja, jb) of one tier from global memory, in order, kU records' loads in flight
template <int TIER, class RecFn>
__device__ __forceinline__ void down_seg_g(RecFn rec, const float *a_sm, int ja, int jb, int d, float (&y)[8]) {
    constexpr int kU = TIER == 0 ? 4 : 8;  // (16 for INT: register spills, measured slower)
    int j = ja;
    for (; j + kU <= jb; j += kU) {
        DownLd<TIER> o[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) down_ldg<TIER>(rec(j + u), d, o[u]);
#pragma unroll
        for (int u = 0; u < kU; u++) down_fma<TIER>(o[u], a_sm[j + u], y);
    }
    for (; j < jb; j++) {
        DownLd<TIER> o;
        down_ldg<TIER>(rec(j), d, o);
        down_fma<TIER>(o, a_sm[j], y);
    }
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

// Pipeline state.  Entries go through the ring in FIFO order; full[s] completes when an
// entry's bytes landed, emptyG / emptyD when its consumers are done (gate/up entry: its P
// units; down entry: every warp).  The three barrier families count their uses separately
// (FfnPipe::nf, ng, nd) so each slot's phase parity is known.
struct FfnShared {
    uint64_t full[kNS];
    uint64_t emptyG[kNS];
    int roff[kNS];          // ring offset of the entry (published before its expect_tx)
    int span[kNS];          // ring bytes the entry holds (incl. wrap waste)
    int pcnt[kNS];          // gate/up parts of a record done (record j -> slot j % kNS)
    float gpart[kNS][kPMax][2];
    int rng[8];             // CTA ranges (6)
};
struct FfnPipe {            // per-CTA counters (registers of the calling kernel, across layers)
    unsigned nf = 0, ng = 0, nd = 0;
};

// thread 0, before any use
__device__ __forceinline__ void ffn_init(FfnShared &sm, int d) {
    for (int i = 0; i < kNS; i++) {
        mbar_init(&sm.full[i], 1);
        mbar_init(&sm.emptyG[i], (uint32_t)kPMax);  // (a record's units arrive kPMax in total)
        sm.pcnt[i] = 0;
    }
    fence_mbar_init();
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar, uint32_t count = 1) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// The FFN over this CTA's n_items records (item j: tier 0 for j < c1, 1 for j < c2, else 2;
// record bytes at global address src(j)).  x must be in xs (fp16, d/8 uint4) before the call
// (the caller's __syncthreads orders it).  pp: this CTA's pipeline counters (persistent
// kernel: carried across layers).  a_sm: [kMaxLocal] floats of smem.  Writes
// partial[blockIdx.x][d]; ends with __syncthreads (the ring is free again).
//  * whole mode (every record fits the ring at once: S7, S13, S70 at P >= 4): warp 0 copies
//    every record (lane j -> record j) before anything else; all warps run phase G on them
//    and phase D reads the down columns from the same copies;
//  * streaming mode (S70H, S70 at P = 2): the last warp is the producer -- it streams the
//    gate/up parts (+ scale/zero tail) of the records through the ring in order, re-using an
//    entry as soon as its P units have arrived on it, then the down parts (+ tail); phase G
//    runs on the other warps; in phase D every warp consumes the down entries in order and the
//    producer re-issues freed space until every down entry is in.
struct NoWait {
    __device__ __forceinline__ void operator()(int) const {}
};
// WaitFn wait(j): called by the lane that issues record j's copies, before them (the LRU
// engine's miss FFN: the record is still landing in the staging area, k_fill publishes a
// per-record flag; everything else: NoWait)
template <class SrcFn, class WaitFn = NoWait>
__device__ __forceinline__ void ffn_run(const FfnArgs &a, int d, int act, int n_items, int c1, int c2,
                                        SrcFn src, uint8_t *ring, const uint4 *xs, float *a_sm,
                                        FfnShared &sm, FfnPipe &pp, float *partial,
                                        unsigned long long *stamps = nullptr, WaitFn wait = WaitFn()) {
    const int NW = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto tier_of = [&](int j) { return j < c1 ? 0 : (j < c2 ? 1 : 2); };
    auto Dof = [&](int t) { return t == 0 ? 2 * d : (t == 1 ? d : d / 2); };
    const int total = c1 * a.nb[0] + (c2 - c1) * a.nb[1] + (n_items - c2) * a.nb[2];
    const bool whole = (n_items <= kNS && total <= kRing) || NW == 1;
    M2C_CHECK(n_items >= 0 && n_items <= kMaxLocal && c1 >= 0 && c1 <= c2 && c2 <= n_items);
    M2C_CHECK(!whole || total <= kRing);
    const uint64_t pol = policy_evict_first();
    const unsigned nf0 = pp.nf, ng0 = pp.ng;
    auto fslot = [&](unsigned e) { return (nf0 + e) % kNS; };
    auto fpar = [&](unsigned e) { return ((nf0 + e) / kNS) & 1u; };
    if (whole) {
        // every record at once: warp 0, lane j -> records j, j + 32 (offsets by warp scans)
        if (warp == 0) {
            int base = 0;
            for (int j0 = 0; j0 < n_items; j0 += 32) {
                const int j = j0 + lane;
                const int sz = j < n_items ? a.nb[tier_of(j)] : 0;
                int inc = sz;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                if (j < n_items) {
                    const unsigned s = fslot(j);
                    M2C_CHECK(base + inc <= kRing && src(j) != nullptr);
                    sm.roff[s] = base + inc - sz;
                    if constexpr (std::is_same<WaitFn, NoWait>::value) {
                        mbar_expect_tx(&sm.full[s], (uint32_t)sz);
                        bulk_g2s(ring + base + inc - sz, src(j), (uint32_t)sz, &sm.full[s], pol);
                    }
                }
                base += __shfl_sync(0xffffffffu, inc, 31);
            }
            if constexpr (!std::is_same<WaitFn, NoWait>::value) {
                // records still landing: one lane issues them in order as each is published,
                // so the units of the early ones run while the later ones arrive
                __syncwarp();
                if (lane == 0)
                    for (int j = 0; j < n_items; j++) {
                        const unsigned s = fslot(j);
                        wait(j);
                        mbar_expect_tx(&sm.full[s], (uint32_t)a.nb[tier_of(j)]);
                        bulk_g2s(ring + sm.roff[s], src(j), (uint32_t)a.nb[tier_of(j)], &sm.full[s], pol);
                    }
            }
        }
    } else if (warp == NW - 1) {
        // streaming: the producer warp (decisions warp-uniform, lane 0 issues) streams the
        // gate/up part (+ scale/zero tail) of each record through the ring in order, re-using
        // an entry as soon as its P units have arrived on it; the record's down part is
        // prefetched into L2 right behind (phase D reads it from global memory)
        int head = 0, tail = 0, wpos = 0, used = 0;
        while (head < n_items) {
            const int t = tier_of(head), D = Dof(t), tailb = a.nb[t] - 3 * D;
            const int sz = 2 * D + tailb;
            const bool wrap = wpos + sz > kRing;
            const int need = (wrap ? kRing - wpos : 0) + sz;
            if (used + need <= kRing && head - tail < kNS) {
                const unsigned s = fslot(head);
                const int off = wrap ? 0 : wpos;
                used += need;
                wpos = off + sz;
                if (lane == 0) {
                    const uint8_t *g = src(head);
                    M2C_CHECK(off + sz <= kRing && need <= kRing && g != nullptr);
                    wait(head);
                    sm.roff[s] = off;
                    sm.span[s] = need;
                    mbar_expect_tx(&sm.full[s], (uint32_t)sz);
                    bulk_g2s(ring + off, g, (uint32_t)(2 * D), &sm.full[s], pol);
                    if (tailb) bulk_g2s(ring + off + 2 * D, g + 3 * D, (uint32_t)tailb, &sm.full[s], pol);
                    prefetch_l2(g + 2 * D, (uint32_t)(a.nb[t] - 2 * D));
                }
                head++;
            } else {
                const unsigned s = (ng0 + tail) % kNS;
                mbar_wait(&sm.emptyG[s], ((ng0 + tail) / kNS) & 1u);
                used -= __shfl_sync(0xffffffffu, sm.span[fslot(tail)], 0);
                tail++;
                if (lane == 0) fence_proxy_async();  // consumers' generic reads precede new copies
            }
            __syncwarp();
        }
    }
    if (stamps && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamps[0]));
    // ---- phase G: gate/up units (record j, part q), round-robin over the compute warps ----
    const int NWc = whole ? NW : NW - 1;
    if (warp < NWc) {
        const int P0 = gu_parts(0, d), P1 = gu_parts(1, d), P2 = gu_parts(2, d);
        const int U0 = c1 * P0, U1 = U0 + (c2 - c1) * P1, U = U1 + (n_items - c2) * P2;
        for (int u = warp; u < U; u += NWc) {
            int j, q, t, Pt;
            if (u < U0) { j = u / P0; q = u - j * P0; t = 0; Pt = P0; }
            else if (u < U1) { j = c1 + (u - U0) / P1; q = (u - U0) - (j - c1) * P1; t = 1; Pt = P1; }
            else { j = c2 + (u - U1) / P2; q = (u - U1) - (j - c2) * P2; t = 2; Pt = P2; }
            const unsigned s = fslot(j);
            mbar_wait(&sm.full[s], fpar(j));
            M2C_CHECK(q < Pt && Pt <= kPMax && j < n_items);
            const int D = Dof(t);
            const uint8_t *rec = ring + sm.roff[s];
            float pg, pu;
            gu_unit_any(t, rec, rec + D, rec + (whole ? 3 * D : 2 * D), d, q, xs, pg, pu);
            if (lane == 0) {
                if (Pt == 1) {
                    a_sm[j] = (act == 1) ? fmaxf(pg, 0.f) * pu : pg / (1.f + expf(-pg)) * pu;
                } else {
                    sm.gpart[s][q][0] = pg;
                    sm.gpart[s][q][1] = pu;
                    __threadfence_block();
                    if (atomicAdd(&sm.pcnt[s], 1) == Pt - 1) {  // last part: combine in order
                        __threadfence_block();
                        float g = 0.f, uu = 0.f;
                        for (int k = 0; k < Pt; k++) {
                            g += sm.gpart[s][k][0];
                            uu += sm.gpart[s][k][1];
                        }
                        sm.pcnt[s] = 0;
                        a_sm[j] = (act == 1) ? fmaxf(g, 0.f) * uu : g / (1.f + expf(-g)) * uu;
                    }
                }
            }
            __syncwarp();
            if (!whole && lane == 0) {  // the record's Pt units arrive kPMax in total
                const uint32_t share = kPMax / Pt;
                mbar_arrive(&sm.emptyG[(ng0 + j) % kNS], q < Pt - 1 ? share : kPMax - (Pt - 1) * share);
            }
        }
    }
    __syncthreads();  // every a_j is in a_sm (and the producer is done)
    if (stamps && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamps[1]));
    // ---- phase D: y[8t, 8t+8) += a_j deq(down_j), records in share order -------------------
    float y[8];
#pragma unroll
    for (int i = 0; i < 8; i++) y[i] = 0.f;
    if (whole) {
        for (int j = 0; j < n_items; j++) {
            const int t = tier_of(j), D = Dof(t);
            const uint8_t *rec = ring + sm.roff[fslot(j)];
            const float aj = a_sm[j];
            if (t == 0) down_acc<0>(rec + 2 * D, rec + 3 * D, d, aj, y);
            else if (t == 1) down_acc<1>(rec + 2 * D, rec + 3 * D, d, aj, y);
            else down_acc<2>(rec + 2 * D, rec + 3 * D, d, aj, y);
        }
    } else {
        down_seg_g<0>(src, a_sm, 0, c1, d, y);
        down_seg_g<1>(src, a_sm, c1, c2, d, y);
        down_seg_g<2>(src, a_sm, c2, n_items, d, y);
    }
    float *out = partial + (int64_t)blockIdx.x * d + 8 * threadIdx.x;
    reinterpret_cast<float4 *>(out)[0] = make_float4(y[0], y[1], y[2], y[3]);
    reinterpret_cast<float4 *>(out)[1] = make_float4(y[4], y[5], y[6], y[7]);
    pp.nf += (unsigned)n_items;
    if (!whole) pp.ng += (unsigned)n_items;
    __syncthreads();  // the ring's entries are consumed
}

struct SmemPtrs {
    uint8_t *ring;
    uint4 *xs;
    int *loc;
    float *a;
};
__device__ __forceinline__ SmemPtrs carve(uint8_t *smem) {
    SmemPtrs p;
    p.ring = smem;
    p.xs = reinterpret_cast<uint4 *>(smem + kRing);
    p.loc = reinterpret_cast<int *>(smem + kRing + kXsBytes);
    p.a = reinterpret_cast<float *>(p.loc + kMaxLocal);
    return p;
}

}  // namespace

// balancing weight of one record, in 16-B units: bytes + lambda * 3d weights.  The FFN phase
// is HBM-bound for the GPU as a whole (every CTA's gate/up stream ends together) and its
// per-CTA tail (the down-projection) costs per record, not per byte, so the split is close to
// per-record: lambda 6 / 16 / 48 B per weight measured 584 / 595 / 596 tokens/s at S70H
// (1456 tokens/s at S7 for all three).
constexpr int kLambda = 16;  // (16-B gate/up units: INT lambda 14 / 16 / 18 and FP16 20 A/B'd,
                             // profiles/r02_ffn_variants.txt)
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

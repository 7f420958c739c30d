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
//  * k_ffn_sel (decode path) first derives the FP16/INT8/INT4 tier lists itself, redundantly
//    in every CTA, from the predictor scores and the 4096-bin score histogram k_pred_s left in
//    global memory: exact thresholds via a second-level histogram, ties by ascending id,
//    then warp-ballot classification of 32-id chunks and a block scan over chunks.  Before
//    waiting on its predecessor it prefetches into L2 the records the previous token selected
//    for this layer (~80% of them recur).
#include "m2c_internal.cuh"

namespace m2c {
namespace {

constexpr int kNBMax = 16;   // records per batch
constexpr int kNSlot = 32;   // mbarriers (>= records in flight)
constexpr int kRing = 192 * 1024;
constexpr int kHistBins = 4096;
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

// exclusive block scan of 3 ints per thread; blockDim.x multiple of 32, <= 1024
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

// in-place exclusive scan of cnt[q][3] over q < Q (smem), all threads
__device__ __forceinline__ void scan_chunks(int *cnt, int Q, int *sm) {
    const int T = blockDim.x;
    const int per = (Q + T - 1) / T;
    const int q0 = min(Q, (int)threadIdx.x * per), q1 = min(Q, q0 + per);
    int v[3] = {0, 0, 0}, ex[3], tot[3];
    for (int q = q0; q < q1; q++)
#pragma unroll
        for (int t = 0; t < 3; t++) v[t] += cnt[3 * q + t];
    block_scan3(v, ex, tot, sm);
    for (int q = q0; q < q1; q++)
#pragma unroll
        for (int t = 0; t < 3; t++) {
            const int c = cnt[3 * q + t];
            cnt[3 * q + t] = ex[t];
            ex[t] += c;
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
    float a_sm[kNBMax];
    int ut[kNBMax][32];  // unit table: [nb-1][warp] -> b | p << 8 | P << 16 (-1: idle)
    int cb[5][5];        // chunk bounds: cb[P][p] = nchunk * p / P
    int rng[8];          // CTA ranges (6)
    int nbatch;
    int scan[96];
    int selv[16];
};

// The FFN main loop over this CTA's n_items records; item j -> global record pointer src(j)
template <class SrcFn>
__device__ __forceinline__ void ffn_loop(const FfnArgs &a, int d, int act, const __half *x, int n_items,
                                         int c1, int c2, SrcFn src, uint8_t *ring, uint4 *xs,
                                         int *dsc, int *bst, FfnShared &sm, float *partial) {
    const int nwarp = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunk = d / 8;
    // tables: unit mapping per batch size, chunk bounds per split
    for (int i = threadIdx.x; i < kNBMax * 32; i += blockDim.x) {
        const int nb = i / 32 + 1, w = i % 32;
        const int P = nwarp / nb >= 4 ? 4 : (nwarp / nb >= 1 ? nwarp / nb : 1);
        sm.ut[nb - 1][w] = (w < nb * P || nwarp < nb) ? ((w % nb) | ((w / nb) << 8) | (P << 16)) : -1;
    }
    if (threadIdx.x < 25) {
        const int P = threadIdx.x / 5, p = threadIdx.x % 5;
        sm.cb[P][p] = P ? nchunk * p / P : 0;
    }
    // thread 0: batches (consecutive records that fit the ring together, with wrap slack)
    if (threadIdx.x == 0) {
        const int nbA = a.nb[0], nbB = a.nb[1], nbC = a.nb[2];
        const int mx = nbA > nbB ? (nbA > nbC ? nbA : nbC) : (nbB > nbC ? nbB : nbC);
        int nbt = 0;
        for (int j0 = 0; j0 < n_items;) {
            int nb = 0, bytes = 0;
            while (nb < kNBMax && j0 + nb < n_items) {
                const int j = j0 + nb;
                const int sz = j < c1 ? nbA : (j < c2 ? nbB : nbC);
                if (nb > 0 && bytes + sz + mx > kRing) break;
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
    int issued = 0, pos_issue = 0, used = 0;
    const uint64_t pol = policy_evict_first();
    auto issue_more = [&](int consumed) {
        while (issued < n_items && issued - consumed < kNSlot) {
            const int j = issued;
            const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
            const int sz = t == 0 ? a.nb[0] : (t == 1 ? a.nb[1] : a.nb[2]);
            const int waste = (pos_issue + sz > kRing) ? kRing - pos_issue : 0;
            if (used + waste + sz > kRing) break;
            const int off = waste ? 0 : pos_issue;
            sm.span[j % kNSlot] = waste + sz;
            used += waste + sz;
            pos_issue = off + sz;
            dsc[j] = off | (t << 24);
            uint64_t *bar = &sm.bars[j % kNSlot];
            mbar_expect_tx(bar, (uint32_t)sz);  // release: dsc[j] is visible to its waiters
            bulk_g2s(ring + off, src(j), (uint32_t)sz, bar, pol);
            issued++;
        }
    };
    if (threadIdx.x == 0) {
        fence_proxy_async();
        issue_more(0);
    }
    // x -> smem as fp16 (read by the warp-local dot products)
    for (int c = threadIdx.x; c < nchunk; c += blockDim.x) xs[c] = reinterpret_cast<const uint4 *>(x)[c];
    __syncthreads();

    float y[8];
#pragma unroll
    for (int i = 0; i < 8; i++) y[i] = 0.f;
    const int nbt = sm.nbatch;
    for (int bi = 0; bi < nbt; bi++) {
        const int j0 = bst[bi], nb = bst[bi + 1] - j0;
        // gate/up: this warp's units (b, p) of the batch
        int P = 1;
        for (int w = warp; w < 32 * ((nb + 31) / 32) && w < (nb > nwarp ? nb : nwarp); w += nwarp) {
            const int u = nb <= nwarp ? sm.ut[nb - 1][w] : (w | (1 << 16));
            if (u < 0) break;
            const int b = u & 0xff, p = (u >> 8) & 0xff;
            P = u >> 16;
            const int j = j0 + b;
            mbar_wait(&sm.bars[j % kNSlot], (uint32_t)((j / kNSlot) & 1));
            const int ds = dsc[j];
            float pg, pu;
            gu_any(ds >> 24, ring + (ds & 0xffffff), xs, d, sm.cb[P][p], sm.cb[P][p + 1], pg, pu);
            pg = warp_sum_f(pg);
            pu = warp_sum_f(pu);
            if (lane == 0) {
                if (P == 1) {
                    sm.a_sm[b] = (act == 1) ? fmaxf(pg, 0.f) * pu : pg / (1.f + expf(-pg)) * pu;
                } else {
                    sm.part[b][p][0] = pg;
                    sm.part[b][p][1] = pu;
                }
            }
        }
        P = nb <= nwarp ? (sm.ut[nb - 1][0] >> 16) : 1;
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
        for (int b = 0; b < nb; b++) {
            const int ds = dsc[j0 + b];
            down_any(ds >> 24, ring + (ds & 0xffffff), d, sm.a_sm[b], y);
        }
        __syncthreads();  // the batch's records are consumed; a_sm/part reusable
        if (threadIdx.x == 0) {
            for (int b = 0; b < nb; b++) used -= sm.span[(j0 + b) % kNSlot];
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

// ---- list-driven FFN (API path: m2c_sparse_ffn_forward, LRU hits / misses) --------------
__global__ void __launch_bounds__(1024, 1)
    k_ffn(FfnArgs a, int d, int act, const __half *__restrict__ x, const int32_t *__restrict__ items,
          const int32_t *__restrict__ counts, float *__restrict__ partial) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    const SmemPtrs S = carve(smem);
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
    ffn_loop(a, d, act, x, n_items, c1, c2, src, S.ring, S.xs, S.dsc, S.bst, sm, partial);
}

// ---- decode path: select (tier lists from scores + histogram) fused with the FFN ----------
__global__ void __launch_bounds__(1024, 1)
    k_ffn_sel(FfnArgs a, SelArgs s, int d, int act, const __half *__restrict__ x,
              float *__restrict__ partial) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    const SmemPtrs S = carve(smem);
    // select scratch inside the ring (unused until the records are requested):
    // hist[4096] | sub[3][2^sh] | cnt[Q][3] | scores[F_r]
    int *hist = reinterpret_cast<int *>(S.ring);
    int *sub = hist + kHistBins;
    const int nsub = 1 << s.sh;
    const int Q = (s.F_r + 31) / 32;
    int *cnt = sub + 3 * nsub;
    int *sc = cnt + 3 * Q;
    const int T = blockDim.x, tid = threadIdx.x;
    const int nwarp = T >> 5, warp = tid >> 5, lane = tid & 31;
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
    if (warp == nwarp - 1 && s.prev_ids) {
        for (int j = lane; j < n_items; j += 32) {
            int t, id;
            if (j < c1) { t = 0; id = s.prev_ids[a0 + j]; }
            else if (j < c2) { t = 1; id = s.prev_ids[n0 + a1 + (j - c1)]; }
            else { t = 2; id = s.prev_ids[n0 + n1 + a2 + (j - c2)]; }
            if (id >= 0 && id < s.F_r) prefetch_l2(a.pool[t] + (int64_t)id * a.nb[t], (uint32_t)a.nb[t]);
        }
    }
    griddep_launch();
    griddep_wait();

    // ---- 0. stage the scores (coalesced) and the histogram ----
    for (int n = tid; n < s.F_r; n += T) sc[n] = s.scores[n] + s.smax;  // biased, >= 0
    const int tg0 = s.k16, tg1 = s.k16 + s.k8, tg2 = s.k;
    const int BPT = (kHistBins + T - 1) / T;
    int lsum = 0;
    for (int i = 0; i < BPT; i++) {  // descending bins: thread t covers [4095 - t*BPT - i]
        const int b = kHistBins - 1 - (tid * BPT + i);
        if (b < 0) break;
        const int v = s.hist[b];
        hist[b] = v;
        lsum += v;
    }
    // ---- 1. bin holding the target-th largest, for the three targets ----
    {
        const int vv[3] = {lsum, 0, 0};
        int ex[3], tot[3];
        block_scan3(vv, ex, tot, sm.scan);
        int cum = ex[0];
        for (int i = 0; i < BPT; i++) {
            const int b = kHistBins - 1 - (tid * BPT + i);
            if (b < 0) break;
            const int v = hist[b];
            if (tg0 > 0 && cum < tg0 && cum + v >= tg0) { sm.selv[0] = b; sm.selv[3] = cum; }
            if (tg1 > 0 && cum < tg1 && cum + v >= tg1) { sm.selv[1] = b; sm.selv[4] = cum; }
            if (tg2 > 0 && cum < tg2 && cum + v >= tg2) { sm.selv[2] = b; sm.selv[5] = cum; }
            cum += v;
        }
    }
    for (int i = tid; i < 3 * nsub; i += T) sub[i] = 0;
    __syncthreads();
    const int bin0 = tg0 > 0 ? sm.selv[0] : -1, bin1 = tg1 > 0 ? sm.selv[1] : -1,
              bin2 = tg2 > 0 ? sm.selv[2] : -1;
    // ---- 2. second level: exact values inside the chosen bins ----
    for (int n = tid; n < s.F_r; n += T) {
        const int v = sc[n];
        const int b = v >> s.sh, lo = v & (nsub - 1);
        if (b == bin0) atomicAdd(&sub[lo], 1);
        if (b == bin1) atomicAdd(&sub[nsub + lo], 1);
        if (b == bin2) atomicAdd(&sub[2 * nsub + lo], 1);
    }
    __syncthreads();
    for (int t = warp; t < 3; t += nwarp) {  // warp t scans sub[t] from the top
        const int tg = t == 0 ? tg0 : (t == 1 ? tg1 : tg2);
        if (tg <= 0) continue;
        const int need = tg - sm.selv[3 + t], bin = sm.selv[t];
        const int per = nsub / 32;
        const int *st = sub + t * nsub;
        int loc_sum = 0;
        for (int i = 0; i < per; i++) loc_sum += st[nsub - 1 - (lane * per + i)];
        int inc = loc_sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y2 = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y2;
        }
        const int excl = inc - loc_sum;
        if (excl < need && inc >= need) {
            int cum = excl;
            for (int i = 0; i < per; i++) {
                const int c = nsub - 1 - (lane * per + i);
                const int v = st[c];
                if (cum + v >= need) {
                    sm.selv[6 + t] = (bin << s.sh) | c;  // exact biased value V_t
                    sm.selv[9 + t] = need - cum;         // how many equal to V_t are in
                    sm.selv[12 + t] = v;                 // how many equal to V_t exist
                    break;
                }
                cum += v;
            }
        }
    }
    __syncthreads();
    const int V0 = tg0 > 0 ? sm.selv[6] : 0x7fffffff, V1 = tg1 > 0 ? sm.selv[7] : 0x7fffffff,
              V2 = tg2 > 0 ? sm.selv[8] : 0x7fffffff;
    const int R0 = tg0 > 0 ? sm.selv[9] : 0, R1 = tg1 > 0 ? sm.selv[10] : 0, R2 = tg2 > 0 ? sm.selv[11] : 0;
    const bool tie = (tg0 > 0 && R0 < sm.selv[12]) || (tg1 > 0 && R1 < sm.selv[13]) ||
                     (tg2 > 0 && R2 < sm.selv[14]);
    const unsigned lt_mask = (1u << lane) - 1u;
    // ---- 3a. (only with partial ties) equal-key ranks in id order: per-chunk counts ----
    if (tie) {
        for (int q = warp; q < Q; q += nwarp) {
            const int n = 32 * q + lane;
            const int v = n < s.F_r ? sc[n] : -1;
            const unsigned e0 = __ballot_sync(0xffffffffu, v == V0), e1 = __ballot_sync(0xffffffffu, v == V1),
                           e2 = __ballot_sync(0xffffffffu, v == V2);
            if (lane == 0) {
                cnt[3 * q] = __popc(e0);
                cnt[3 * q + 1] = __popc(e1);
                cnt[3 * q + 2] = __popc(e2);
            }
        }
        __syncthreads();
        scan_chunks(cnt, Q, sm.scan);
    }
    // tier of element n (lane of chunk q); `eq` holds the chunk's equal-key prefix (if tie)
    auto tier_at = [&](int v, int q) -> int {
        bool in0 = v > V0, in1 = v > V1, in2 = v > V2;
        if (tie) {
            const unsigned e0 = __ballot_sync(0xffffffffu, v == V0), e1 = __ballot_sync(0xffffffffu, v == V1),
                           e2 = __ballot_sync(0xffffffffu, v == V2);
            if (v == V0) in0 = cnt[3 * q] + __popc(e0 & lt_mask) < R0;
            if (v == V1) in1 = cnt[3 * q + 1] + __popc(e1 & lt_mask) < R1;
            if (v == V2) in2 = cnt[3 * q + 2] + __popc(e2 & lt_mask) < R2;
        } else {
            in0 = in0 || v == V0;
            in1 = in1 || v == V1;
            in2 = in2 || v == V2;
        }
        return in0 ? 0 : (in1 ? 1 : (in2 ? 2 : -1));
    };
    // ---- 3b. tier membership per 32-id chunk (ballots) -> positions by a scan over chunks ----
    int *tcnt = tie ? sc + s.F_r : cnt;  // keep the eq prefixes if needed: second table after sc
    for (int q = warp; q < Q; q += nwarp) {
        const int n = 32 * q + lane;
        const int v = n < s.F_r ? sc[n] : -1;
        const int tr = tier_at(v, q);
        const unsigned m0 = __ballot_sync(0xffffffffu, tr == 0), m1 = __ballot_sync(0xffffffffu, tr == 1),
                       m2 = __ballot_sync(0xffffffffu, tr == 2);
        if (lane == 0) {
            tcnt[3 * q] = __popc(m0);
            tcnt[3 * q + 1] = __popc(m1);
            tcnt[3 * q + 2] = __popc(m2);
        }
    }
    __syncthreads();
    scan_chunks(tcnt, Q, sm.scan);
    // ---- 3c. emit: this CTA's records into loc[], CTA 0 the whole lists ----
    const int lo0 = a0, hi0 = a0 + c1, lo1 = a1, hi1 = a1 + (c2 - c1), lo2 = a2, hi2 = a2 + (n_items - c2);
    for (int q = warp; q < Q; q += nwarp) {
        const int b0 = tcnt[3 * q], b1 = tcnt[3 * q + 1], b2 = tcnt[3 * q + 2];
        const int e0n = q + 1 < Q ? tcnt[3 * q + 3] : s.k16, e1n = q + 1 < Q ? tcnt[3 * q + 4] : s.k8,
                  e2n = q + 1 < Q ? tcnt[3 * q + 5] : n2;
        const bool mine = (b0 < hi0 && e0n > lo0) || (b1 < hi1 && e1n > lo1) || (b2 < hi2 && e2n > lo2);
        if (!mine && !(blockIdx.x == 0 && s.out_ids)) continue;
        const int n = 32 * q + lane;
        const int v = n < s.F_r ? sc[n] : -1;
        const int tr = tier_at(v, q);
        const unsigned m0 = __ballot_sync(0xffffffffu, tr == 0), m1 = __ballot_sync(0xffffffffu, tr == 1),
                       m2 = __ballot_sync(0xffffffffu, tr == 2);
        if (tr >= 0) {
            const unsigned m = tr == 0 ? m0 : (tr == 1 ? m1 : m2);
            const int p = (tr == 0 ? b0 : (tr == 1 ? b1 : b2)) + __popc(m & lt_mask);
            const int lo = tr == 0 ? lo0 : (tr == 1 ? lo1 : lo2), hi = tr == 0 ? hi0 : (tr == 1 ? hi1 : hi2);
            const int lb = tr == 0 ? 0 : (tr == 1 ? c1 : c2);
            if (p >= lo && p < hi) S.loc[lb + p - lo] = n;
            if (blockIdx.x == 0 && s.out_ids) s.out_ids[(tr == 0 ? 0 : (tr == 1 ? n0 : n0 + n1)) + p] = n;
        }
    }
    __syncthreads();
    auto src = [&](int j) -> const uint8_t * {
        const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
        return a.pool[t] + (int64_t)S.loc[j] * a.nb[t];
    };
    ffn_loop(a, d, act, x, n_items, c1, c2, src, S.ring, S.xs, S.dsc, S.bst, sm, partial);
}

}  // namespace

cudaError_t init_ffn_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_ffn_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
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
    cudaError_t e = launch_k(k_ffn, dim3(c->G), dim3(d / 8), kSmemBytes, st, a, d, c->desc.act, x,
                             items, counts, partial);
    c->launch_counter++;
    return e;
}

bool ffn_sel_supported(m2c_ctx *c, const m2c_tier_plan &p) {
    // every CTA's share must fit the local item list; select scratch must fit the ring
    FfnArgs a;
    LayerState dummy;
    fill_args(c, dummy, p, a);
    const long long W = (long long)p.k_fp16 * a.wt[0] + (long long)p.k_int8 * a.wt[1] + (long long)p.k_int4 * a.wt[2];
    const long long per = W / c->G + 1;
    const int wmin = a.wt[2] < a.wt[1] ? (a.wt[2] < a.wt[0] ? a.wt[2] : a.wt[0]) : (a.wt[1] < a.wt[0] ? a.wt[1] : a.wt[0]);
    const long long Q = (c->F_r + 31) / 32;
    const long long scratch = 4LL * (kHistBins + 3 * (1LL << c->sel_sh) + 6 * Q + 2LL * c->F_r);
    return per / wmin + 3 <= kMaxLocal && c->sel_sh <= 12 && scratch <= kRing;
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
    cudaError_t e = launch_k(k_ffn_sel, dim3(c->G), dim3(d / 8), kSmemBytes, st, a, s, d, c->desc.act,
                             x, partial);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

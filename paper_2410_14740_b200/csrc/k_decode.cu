// k_decode.cu -- the persistent decode kernel: ONE cooperative launch runs a whole token
// through every layer of the resident stack (a1 -> a7 of SURVEY §8, per layer).
//
// Why: batch-1 decode of the sparse FFN moves ~17 MB per layer (S7), i.e. ~2.7 us at HBM
// speed, while a chain of five dependent kernels per layer costs ~40 us of launch / drain /
// ramp latency (profiles/).  Here one CTA per SM stays resident for the whole token and the
// phases of a layer are separated by grid barriers (~0.5 us each) instead of kernel
// boundaries:
//   P1  x -> xq = Q(x) (every CTA, from L2), h = A xq for this CTA's rows of A   [a1]
//   --- barrier
//   P2  hq = Q(h) (every CTA), scores s = B hq for this CTA's neurons, 4096-bin
//       histogram of s (global atomics)                                          [a2]
//   --- barrier
//   P3  every CTA derives the three rank cuts itself (histogram scan, exact refinement of
//       the cut bins, ties by id -- R3), classifies ALL neurons from a shared-memory copy of
//       the scores and takes its byte-balanced share of the tier lists (no barrier needed:
//       the lists are a pure function of s)                                       [a3]
//   P4  fused dequant-GEMV FFN over the share (ffn_dev.cuh, same code as k_ffn) -> partial y
//                                                                                 [a6]
//   --- barrier
//   P5  fixed-order reduction of the partials (the k_reduce order) for this CTA's 32-column
//       chunks, x_{l+1} = fp16(x + fp16(y)) (R14)                                 [a7]
//   --- barrier
// While layer l runs, every CTA streams its share of layer l+1's predictor slices and of the
// records the previous token selected for layer l+1 (~80% recur) into L2, so the FFN's
// TMA reads mostly hit L2 (cross-layer lookahead in hardware terms).
// Results are bit-identical to the per-phase kernel chain (same select rule, same per-CTA FFN
// shares and batches, same reduction order): tests/test_gpu_parity.py checks it.
#include <cstdlib>

#include "ffn_dev.cuh"

namespace m2c {
namespace {

constexpr int kBins = 4096;
// profiling stamps per (layer, CTA): 0 layer start, 1 P1 done, 2 after B1, 3 P2 done, 4 after
// B2, 5 P3 done, 6 P4 done, 7 after B4, 8 P5 done, 9 kernel end (last layer only); P3 steps:
// 10 cuts exact, 11 own neurons classified + published, 12 after barrier 3, 13 list share
// gathered.  (Publishing the counts as tagged words polled by every CTA instead of barrier 3
// measured slower: 148 x 148 pollers on ten cache lines.)
constexpr int kStamps = kDecodeStamps;
constexpr int kBucket = 32;       // (score, id) pairs kept per histogram bin
constexpr int kCoarse = 64;       // coarse bins (64 fine bins each)
// ring-aliased scratch of P1..P3 (bytes): xq [0, 8K) | hq [8K, 8.5K) | own scores | from 32K:
// histogram (P3a), all scores (degenerate-tie fallback), per-CTA counts (P3b)
constexpr int kOwnOff = 9216;     // <= 4096 ints: this CTA's scores
constexpr int kSbufOff = 32768;   // [F_r] ints

struct DecLayer {
    const int8_t *A, *B;
    const uint8_t *pool[3];
};

struct DecArgs {
    const DecLayer *layers;
    int n_layers, d, r, F_r, act;
    int k16, k8, k4;
    int smax, sh;
    int nb[3], wt[3];
    __half *x;                  // [d] in/out
    int32_t *h;                 // [r]
    int32_t *s;                 // [F_r]
    int *ghist;                 // [2][4096]
    int32_t *lists;             // [n_layers][max(k,1)]  (the tier lists; next token's prefetch hint)
    float *partial;             // [G][d]
    unsigned *bar_flags;        // [32]: [0] = grid-barrier arrival counter
    unsigned *bar_epoch;
    uint32_t *err;
    unsigned long long *prof;   // [n_layers][G][kStamps] globaltimer stamps, or null
    int prefetch;
    int2 *bucket;               // [2][4096][kBucket] (score, id) per bin (layer parity)
    int *stage;                 // [3][G][ceil(F_r / G)] per-CTA compacted selected ids
    int *ccount;                // [G][4] per-CTA tier counts
    int *bin_sh;                // [n_layers] histogram scale per layer (adapted token to token)
    unsigned *sabs;             // [G] per-CTA max |s| of the current layer
};

// histogram bin of a raw score: monotone, clamped; 2^sh-wide bins centred on 0
__device__ __forceinline__ int bin_of(int s, int sh) { return min(max((s >> sh) + 2048, 0), 4095); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier #target (counted across launches): every CTA adds 1 to one counter with a
// release reduction; thread 0 polls it with acquire loads until it reaches target * G
// (wrap-safe).  Measured ~1.4 us on B200 (tools/mb_gridsync.cu: per-CTA flag words polled
// by a warp cost ~3 us).  Warp 1 runs `work` (latency-tolerant side work) meanwhile.  A 2 s
// timeout sets err bit 4 instead of hanging the GPU.
template <class F>
__device__ __forceinline__ void grid_sync(unsigned *counter, unsigned target, uint32_t *err, F work) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockDim.x == 32) work();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
        const unsigned want = target * gridDim.x;
        const unsigned long long t0 = gtimer();
        while ((int)(ld_acquire(counter) - want) < 0) {
            if (gtimer() - t0 > 2000000000ull) {
                atomicOr(err, 4u);
                break;
            }
        }
    } else if (threadIdx.x >= 32 && threadIdx.x < 64) {
        work();  // warp 1: e.g. L2 prefetch while thread 0 waits
    }
    __syncthreads();
}
__device__ __forceinline__ void grid_sync(unsigned *flags, unsigned target, uint32_t *err) {
    grid_sync(flags, target, err, [] {});
}

__device__ __forceinline__ int block_max_u(unsigned v, unsigned *sm32) {
    v = __reduce_max_sync(0xffffffffu, v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sm32[warp] = v;
    __syncthreads();
    return (int)__reduce_max_sync(0xffffffffu, lane < nw ? sm32[lane] : 0u);
}
__device__ __forceinline__ int block_sum(int v, int *sm32) {
    v = __reduce_add_sync(0xffffffffu, v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sm32[warp] = v;
    __syncthreads();
    return __reduce_add_sync(0xffffffffu, lane < nw ? sm32[lane] : 0);
}
// exclusive block scan of 3 ints (any blockDim multiple of 32, <= 1024); totals in tot
__device__ __forceinline__ void block_exscan3(const int v[3], int ex[3], int tot[3], int *sm /*[3][32]*/) {
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

__device__ __forceinline__ int q127_f32(float a, float M, float inv) {  // a = |v| >= 0, M > 0
    int q = (int)fmaf(a, inv, 0.5f);
    const float a254 = 254.f * a;
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

// L2 prefetch of layer lj's predictor slices of this CTA and its share of the records the
// previous token selected for lj (one warp, fire and forget)
__device__ __forceinline__ void prefetch_layer(const DecArgs &p, int lj) {
    if (p.prefetch == 0) return;
    const DecLayer Lj = p.layers[lj];
    const int lane = threadIdx.x & 31, G = gridDim.x, cta = blockIdx.x;
    const int rph = (p.r + G - 1) / G, rps = (p.F_r + G - 1) / G;
    if (lane < rph && cta * rph + lane < p.r)
        prefetch_l2(Lj.A + (int64_t)(cta * rph + lane) * p.d, (uint32_t)p.d);
    {
        const int n0 = cta * rps, n1 = min(p.F_r, n0 + rps);
        for (int n = n0 + lane * 64; n < n1; n += 32 * 64)  // <= 64 rows (16 KB at r = 256) per call
            prefetch_l2(Lj.B + (int64_t)n * p.r, (uint32_t)(min(64, n1 - n) * p.r));
    }
    if (p.prefetch == 1) {
        const int k = p.k16 + p.k8 + p.k4;
        const int32_t *ids = p.lists + (int64_t)lj * (k > 0 ? k : 1);
        const int i0 = (int)((long long)k * cta / G), i1 = (int)((long long)k * (cta + 1) / G);
        for (int i = i0 + lane; i < i1; i += 32) {
            const int t = i < p.k16 ? 0 : (i < p.k16 + p.k8 ? 1 : 2);
            const int id = __ldcg(ids + i);
            if (id >= 0 && id < p.F_r) prefetch_l2(Lj.pool[t] + (int64_t)id * p.nb[t], (uint32_t)p.nb[t]);
        }
    }
}

template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_decode(DecArgs p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    __shared__ FfnArgs fa;
    __shared__ unsigned red_u[32];
    __shared__ int red_i[32];
    __shared__ int scan_sm[96];
    __shared__ int cut_bin[3], cut_need[3], cut_V[3], cut_I[3], ncand[3];
    const SmemPtrs S = carve(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5, G = gridDim.x, cta = blockIdx.x;
    const int d = p.d, r = p.r, F_r = p.F_r;
    const int kk = p.k16 + p.k8 + p.k4;
    const int tg[3] = {p.k16, p.k16 + p.k8, kk};
    if (tid == 0) {
        for (int i = 0; i < kNSlot; i++) mbar_init(&sm.bars[i], 1);
        fence_mbar_init();
        for (int t = 0; t < 3; t++) {
            fa.nb[t] = p.nb[t];
            fa.wt[t] = p.wt[t];
        }
        fa.seg[0] = 0;
        fa.seg[1] = p.k16;
        fa.seg[2] = p.k16 + p.k8;
        int rg[6];  // this CTA's FFN share of each tier list: the same for every layer
        cta_ranges(fa, p.k16, p.k8, p.k4, cta, G, rg);
        for (int i = 0; i < 6; i++) sm.rng[i] = rg[i];
    }
    ffn_tables(sm, d);
    const unsigned base = ld_relaxed(p.bar_epoch);  // read by every CTA before its first arrival
    unsigned nbar = 0;
    unsigned jb = 0;  // mbarrier uses of this CTA so far
    // per-CTA globaltimer stamps (profiling): [l][cta][kStamps], see STAMP below
    unsigned long long *prof0 = (p.prof && tid == 0) ? p.prof + (int64_t)cta * kStamps : nullptr;
    const int64_t prof_layer = (int64_t)G * kStamps;
    unsigned long long *prof = nullptr;
#define STAMP(i) \
    if (prof) prof[i] = gtimer()
    if (warp == NW - 1) prefetch_layer(p, 0);

    for (int l = 0; l < p.n_layers; l++) {
        const DecLayer Ld = p.layers[l];
        int *hist = p.ghist + (l & 1) * kBins;
        int32_t *lst = p.lists + (int64_t)l * (kk > 0 ? kk : 1);
        prof = prof0 ? prof0 + l * prof_layer : nullptr;
        STAMP(0);

        // ================= P1: xq = Q(x), h rows ==================================
        {
            int8_t *xq = reinterpret_cast<int8_t *>(S.ring);
            // this warp's first 16 B of its A row segment, loaded before x (independent of it)
            const int rph = (r + G - 1) / G;
            const int row0 = cta * rph, nrow = max(0, min(rph, r - row0));
            const int wpr = NW >= nrow && nrow > 0 ? NW / nrow : 1;  // warps per row
            const int n16 = d / 16, per = (n16 + wpr - 1) / wpr;
            const int rr_first = warp / wpr, seg = warp % wpr;
            const int c0 = seg * per, c1 = min(n16, c0 + per);
            int4 a_pre = make_int4(0, 0, 0, 0);
            if (rr_first < nrow && c0 + lane < c1)
                a_pre = __ldg(reinterpret_cast<const int4 *>(Ld.A + (int64_t)(row0 + rr_first) * d) + c0 + lane);
            const uint4 xv = __ldcg(reinterpret_cast<const uint4 *>(p.x) + tid);  // NT == d / 8
            S.xs[tid] = xv;
            const unsigned m2 = __vmaxu2(__vmaxu2(xv.x & 0x7fff7fffu, xv.y & 0x7fff7fffu),
                                         __vmaxu2(xv.z & 0x7fff7fffu, xv.w & 0x7fff7fffu));
            unsigned mx = (unsigned)block_max_u(max(m2 & 0xffffu, m2 >> 16), red_u);
            if (mx >= 0x7c00) {  // Inf / NaN: flag, quantise as zero
                if (cta == 0 && tid == 0) atomicOr(p.err, 1u);
                mx = 0;
            }
            const float M = __half2float(__ushort_as_half((unsigned short)mx));
            const float inv = mx ? 127.f / M : 0.f;
            const uint32_t w[4] = {xv.x, xv.y, xv.z, xv.w};
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
            reinterpret_cast<uint2 *>(xq)[tid] = make_uint2(packed[0], packed[1]);
            __syncthreads();
            if (nrow > 0) {
                for (int rr = rr_first; rr < nrow; rr += (NW / wpr > 0 ? NW / wpr : 1)) {
                    const int4 *a4 = reinterpret_cast<const int4 *>(Ld.A + (int64_t)(row0 + rr) * d);
                    const int4 *x4 = reinterpret_cast<const int4 *>(xq);
                    int acc = 0;
                    for (int c = c0 + lane; c < c1; c += 32) {
                        const int4 av = (rr == rr_first && c == c0 + lane) ? a_pre : __ldg(a4 + c);
                        const int4 xw = x4[c];
                        acc = __dp4a(av.x, xw.x, acc);
                        acc = __dp4a(av.y, xw.y, acc);
                        acc = __dp4a(av.z, xw.z, acc);
                        acc = __dp4a(av.w, xw.w, acc);
                    }
                    acc = __reduce_add_sync(0xffffffffu, acc);
                    if (wpr == 1) {
                        if (lane == 0) p.h[row0 + rr] = acc;
                    } else if (lane == 0) {
                        red_i[warp] = acc;
                    }
                }
                if (wpr > 1) {
                    __syncthreads();
                    if (tid < nrow) {
                        int s = 0;
                        for (int w2 = 0; w2 < wpr; w2++) s += red_i[tid * wpr + w2];
                        p.h[row0 + tid] = s;
                    }
                }
            }
        }
        STAMP(1);
        grid_sync(p.bar_flags, base + ++nbar, p.err,
                  [&] { prefetch_layer(p, l + 1 < p.n_layers ? l + 1 : 0); });
        STAMP(2);

        // ================= P2: hq = Q(h), scores, histogram ==========================
        const int shl = __ldcg(p.bin_sh + l);  // this token's histogram scale for layer l
        {
            int8_t *hq = reinterpret_cast<int8_t *>(S.ring) + 8192;
            // lanes per neuron LPN, 16-B chunks per lane CPL (r = 256: 4 x 4; r = 32: 1 x 2)
            const int C16 = r / 16, CPL = C16 >= 4 ? 4 : C16, LPN = C16 / CPL, npw = 32 / LPN;
            const int part = lane % LPN, sub = lane / LPN;
            const int rps = (F_r + G - 1) / G;
            const int n0 = cta * rps, n1 = min(F_r, n0 + rps);
            const int step = NW * npw;
            int nb0 = n0 + warp * npw;
            int4 bv[4];
            auto load_b = [&]() {  // B loads are independent of h: issued first
                const int n = nb0 + sub;
                const int4 *b4 = reinterpret_cast<const int4 *>(Ld.B + (int64_t)n * r) + part * CPL;
#pragma unroll
                for (int c = 0; c < 4; c++) bv[c] = (c < CPL && n < n1) ? __ldg(b4 + c) : make_int4(0, 0, 0, 0);
            };
            load_b();
            int hv0 = tid < r ? __ldcg(p.h + tid) : 0;
            int mh = abs(hv0);
            for (int i = tid + NT; i < r; i += NT) mh = max(mh, abs(__ldcg(p.h + i)));
            mh = block_max_u((unsigned)mh, red_u);
            const double Mh = (double)mh, invh = mh ? 127.0 / Mh : 0.0;
            for (int i = tid; i < r; i += NT) {
                const int hv = i == tid ? hv0 : __ldcg(p.h + i);
                const int q = mh ? q127_f64((double)abs(hv), Mh, invh) : 0;
                hq[i] = (int8_t)(hv < 0 ? -q : q);
            }
            __syncthreads();
            const int4 *hq4 = reinterpret_cast<const int4 *>(hq) + part * CPL;
            unsigned amax = 0;
            int *own = reinterpret_cast<int *>(S.ring + kOwnOff);  // this CTA's scores (P3)
            int2 *bkt = p.bucket + (size_t)(l & 1) * kBins * kBucket;
            while (nb0 < n1) {
                int acc = 0;
#pragma unroll
                for (int c = 0; c < 4; c++)
                    if (c < CPL) {
                        const int4 hv4 = hq4[c];
                        acc = __dp4a(bv[c].x, hv4.x, acc);
                        acc = __dp4a(bv[c].y, hv4.y, acc);
                        acc = __dp4a(bv[c].z, hv4.z, acc);
                        acc = __dp4a(bv[c].w, hv4.w, acc);
                    }
                for (int o = LPN / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                const int n = nb0 + sub;
                if (part == 0 && n < n1) {
                    const int b = bin_of(acc, shl);
                    p.s[n] = acc;
                    own[n - n0] = acc;
                    amax = max(amax, (unsigned)abs(acc));
                    const int slot = atomicAdd(&hist[b], 1);
                    if (slot < kBucket) bkt[(size_t)b * kBucket + slot] = make_int2(acc, n);
                }
                nb0 += step;
                if (nb0 < n1) load_b();
            }
            amax = block_max_u(amax, red_u);  // one plain store per CTA (no same-address atomics)
            if (tid == 0) p.sabs[cta] = amax;
        }
        STAMP(3);
        grid_sync(p.bar_flags, base + ++nbar, p.err);
        STAMP(4);
        // next token's histogram scale for this layer: |s| < 2048 << sh (no clamped bins)
        if (cta == 0 && warp == 0) {
            unsigned m = 0;
            for (int c = lane; c < G; c += 32) m = max(m, __ldcg(p.sabs + c));
            m = __reduce_max_sync(0xffffffffu, m);
            int sh = 0;
            while ((m >> sh) >= 2048u) sh++;
            if (lane == 0) p.bin_sh[l] = sh;
        }
        // the other histogram buffer was last read in layer l-1's P3: clear it for layer l+1
        if (cta == G - 1)
            for (int i = tid; i < kBins; i += NT) p.ghist[((l + 1) & 1) * kBins + i] = 0;

        // ================= P3a: exact cuts (every CTA), classify own neurons, publish ========
        // Cut t (t = 0, 1, 2: the k16-th, (k16+k8)-th and k-th score in (score desc, id asc)
        // order, R3) is found by warp t: suffix scans of the 64 coarse then 64 fine histogram
        // bins locate the bin and the rank needed inside it; the bin's bucket (<= kBucket
        // (score, id) pairs written in P2) is ranked exactly.  An overflowing bucket (massive
        // ties) falls back to block-wide binary searches over all scores.
        {
            const int2 *bkt = p.bucket + (size_t)(l & 1) * kBins * kBucket;
            if (tid < 3) {
                cut_V[tid] = 0x7fffffff;  // empty cut: nothing is above it
                cut_I[tid] = -1;
                cut_bin[tid] = -1;
                ncand[tid] = 0;
            }
            // the histogram -> smem in one round of 16-B loads; coarse sums of 64 bins after it
            int *hs = reinterpret_cast<int *>(S.ring + kSbufOff);
#pragma unroll 4
            for (int i = tid; i < kBins / 4; i += NT)
                reinterpret_cast<int4 *>(hs)[i] = __ldcg(reinterpret_cast<const int4 *>(hist) + i);
            __syncthreads();
            for (int cidx = warp; cidx < kCoarse; cidx += NW) {
                const int v = __reduce_add_sync(0xffffffffu, hs[64 * cidx + lane] + hs[64 * cidx + 32 + lane]);
                if (lane == 0) hs[kBins + cidx] = v;
            }
            __syncthreads();
            for (int t = warp; t < 3; t += NW) {
                if (tg[t] <= 0) continue;
                // coarse: lane covers descending coarse bins 63 - 2 lane, 62 - 2 lane
                const int ca = hs[kBins + 63 - 2 * lane], cb = hs[kBins + 62 - 2 * lane];
                int inc = ca + cb;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                int before = inc - ca - cb;  // count above this lane's first coarse bin
                int cbin = -1, need = 0;
                if (before < tg[t] && before + ca >= tg[t]) {
                    cbin = 63 - 2 * lane;
                    need = tg[t] - before;
                } else if (before + ca < tg[t] && before + ca + cb >= tg[t]) {
                    cbin = 62 - 2 * lane;
                    need = tg[t] - before - ca;
                }
                const unsigned who = __ballot_sync(0xffffffffu, cbin >= 0);
                if (!who) {  // histogram total < target: cannot happen with a consistent plan
                    if (lane == 0) atomicOr(p.err, 8u);
                    continue;
                }
                const int src = __ffs(who) - 1;
                cbin = __shfl_sync(0xffffffffu, cbin, src);
                need = __shfl_sync(0xffffffffu, need, src);
                // fine bins of that coarse bin, descending
                const int fa_ = hs[64 * cbin + 63 - 2 * lane];
                const int fb_ = hs[64 * cbin + 62 - 2 * lane];
                inc = fa_ + fb_;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                before = inc - fa_ - fb_;
                int fbin = -1, fneed = 0, m = 0;
                if (before < need && before + fa_ >= need) {
                    fbin = 64 * cbin + 63 - 2 * lane;
                    fneed = need - before;
                    m = fa_;
                } else if (before + fa_ < need && before + fa_ + fb_ >= need) {
                    fbin = 64 * cbin + 62 - 2 * lane;
                    fneed = need - before - fa_;
                    m = fb_;
                }
                const int src2 = __ffs(__ballot_sync(0xffffffffu, fbin >= 0)) - 1;
                fbin = __shfl_sync(0xffffffffu, fbin, src2);
                fneed = __shfl_sync(0xffffffffu, fneed, src2);
                m = __shfl_sync(0xffffffffu, m, src2);
                if (lane == 0) {
                    cut_bin[t] = fbin;
                    cut_need[t] = fneed;
                    ncand[t] = m;
                }
                if (m <= kBucket) {  // exact rank of the bucket's pairs: the fneed-th is the cut
                    const int2 ci = lane < m ? __ldcg(bkt + (size_t)fbin * kBucket + lane) : make_int2(0, 0);
                    int rank = 0;
                    for (int j = 0; j < m; j++) {
                        const int vj = __shfl_sync(0xffffffffu, ci.x, j), nj = __shfl_sync(0xffffffffu, ci.y, j);
                        rank += (vj > ci.x) || (vj == ci.x && nj < ci.y);
                    }
                    if (lane < m && rank == fneed - 1) {
                        cut_V[t] = ci.x;
                        cut_I[t] = ci.y;
                    }
                }
            }
            __syncthreads();
            if ((tg[0] > 0 && ncand[0] > kBucket) || (tg[1] > 0 && ncand[1] > kBucket) ||
                (tg[2] > 0 && ncand[2] > kBucket)) {
                // degenerate: all scores -> smem, binary searches with block-wide counts
                int *sbuf = reinterpret_cast<int *>(S.ring + kSbufOff);
                for (int n = tid; n < F_r; n += NT) sbuf[n] = __ldcg(p.s + n);
                __syncthreads();
                for (int t = 0; t < 3; t++) {
                    if (tg[t] <= 0 || ncand[t] <= kBucket) continue;
                    int lo = -p.smax, hi = p.smax;
                    while (lo < hi) {  // largest V with #{s >= V} >= tg
                        const int mid = lo + (hi - lo + 1) / 2;
                        int c = 0;
                        for (int n = tid; n < F_r; n += NT) c += sbuf[n] >= mid;
                        if (block_sum(c, red_i) >= tg[t]) lo = mid;
                        else hi = mid - 1;
                    }
                    const int V = lo;
                    int c = 0;
                    for (int n = tid; n < F_r; n += NT) c += sbuf[n] > V;
                    const int R = tg[t] - block_sum(c, red_i);
                    int ilo = 0, ihi = F_r - 1;
                    while (ilo < ihi) {  // smallest I with #{n <= I : s == V} >= R
                        const int mid = (ilo + ihi) >> 1;
                        int c2_ = 0;
                        for (int n = tid; n <= mid; n += NT) c2_ += sbuf[n] == V;
                        if (block_sum(c2_, red_i) >= R) ihi = mid;
                        else ilo = mid + 1;
                    }
                    if (tid == 0) {
                        cut_V[t] = V;
                        cut_I[t] = ilo;
                    }
                    __syncthreads();
                }
            }
            STAMP(10);
            // classify this CTA's own neurons (P2's block, scores kept in smem); compact the
            // selected ids of each tier in id order into this CTA's staging row
            const int V0 = cut_V[0], V1 = cut_V[1], V2 = cut_V[2];
            const int I0 = cut_I[0], I1 = cut_I[1], I2 = cut_I[2];
            const int *own = reinterpret_cast<const int *>(S.ring + kOwnOff);
            const int rps = (F_r + G - 1) / G;
            const int n0 = cta * rps, nown = max(0, min(rps, F_r - n0));
            int code = 3;
            if (tid < nown) {
                const int v = own[tid], n = n0 + tid;
                const int a0 = (v > V0) | ((v == V0) & (n <= I0));
                const int a1 = (v > V1) | ((v == V1) & (n <= I1));
                const int a2 = (v > V2) | ((v == V2) & (n <= I2));
                code = 3 - a0 - a1 - a2;  // nested cuts
            }
            const unsigned lt = (1u << lane) - 1u;
            unsigned bal[3];
#pragma unroll
            for (int t = 0; t < 3; t++) bal[t] = __ballot_sync(0xffffffffu, code == t);
            if (lane == 0)
#pragma unroll
                for (int t = 0; t < 3; t++) scan_sm[t * 32 + warp] = __popc(bal[t]);
            __syncthreads();
            if (code < 3) {
                int pos = __popc(bal[code] & lt);
                for (int w = 0; w < warp; w++) pos += scan_sm[code * 32 + w];
                p.stage[((size_t)code * G + cta) * rps + pos] = n0 + tid;
            }
            if (tid < 3) {
                int c = 0;
                for (int w = 0; w < NW; w++) c += scan_sm[tid * 32 + w];
                p.ccount[cta * 4 + tid] = c;
            }
        }
        STAMP(11);
        grid_sync(p.bar_flags, base + ++nbar, p.err);
        STAMP(12);

        // ================= P3b: this CTA's share of the tier lists ============================
        int n_items, c1, c2;
        {
            // thread-contiguous source CTAs: their counts (one 16-B load each), a block scan of
            // the three tier counts -> each source's list offsets; every thread copies the part of
            // its sources' ids that falls into this CTA's share [lo_t, hi_t)
            constexpr int kMaxCPT = 5;  // G <= 160, blockDim >= 32
            const int CPT = (G + NT - 1) / NT;
            const int cA = min(G, tid * CPT), cB = min(G, cA + CPT);
            int4 *cc = reinterpret_cast<int4 *>(S.ring + kSbufOff);  // this thread's sources' counts
            int sum3[3] = {0, 0, 0};
#pragma unroll
            for (int k = 0; k < kMaxCPT; k++) {
                const int4 q = (k < CPT && cA + k < cB) ? __ldcg(reinterpret_cast<const int4 *>(p.ccount) + cA + k)
                                                        : make_int4(0, 0, 0, 0);
                if (k < CPT && cA + k < cB) cc[cA + k] = q;
                sum3[0] += q.x;
                sum3[1] += q.y;
                sum3[2] += q.z;
            }            int ex[3], tot[3];
            block_exscan3(sum3, ex, tot, scan_sm);
            int rg[6];
#pragma unroll
            for (int i = 0; i < 6; i++) rg[i] = sm.rng[i];
            const int off1 = rg[1] - rg[0], off2 = off1 + rg[3] - rg[2];
            c1 = off1;
            c2 = off2;
            n_items = off2 + rg[5] - rg[4];
            const int rps = (F_r + G - 1) / G;
            const int offs[3] = {0, off1, off2};
            const int segs[3] = {0, p.k16, p.k16 + p.k8};
#pragma unroll
            for (int k = 0; k < kMaxCPT; k++) {
                if (k >= CPT || cA + k >= cB) break;
                const int c = cA + k;
                const int4 q = cc[c];
                const int cnt[3] = {q.x, q.y, q.z};
#pragma unroll
                for (int t = 0; t < 3; t++) {
                    const int s0 = ex[t];
                    ex[t] += cnt[t];
                    const int a = max(rg[2 * t], s0), b = min(rg[2 * t + 1], s0 + cnt[t]);
                    const int *src = p.stage + ((size_t)t * G + c) * rps - s0;
                    for (int pos0 = a; pos0 < b; pos0 += 8) {
                        int ids[8];
#pragma unroll
                        for (int u = 0; u < 8; u++) ids[u] = pos0 + u < b ? __ldcg(src + pos0 + u) : 0;
#pragma unroll
                        for (int u = 0; u < 8; u++)
                            if (pos0 + u < b) {
                                S.loc[offs[t] + pos0 + u - rg[2 * t]] = ids[u];
                                lst[segs[t] + pos0 + u] = ids[u];
                            }
                    }
                }
            }
            if (tid == 0) {
                if (tot[0] != p.k16 || tot[1] != p.k8 || tot[2] != p.k4) atomicOr(p.err, 8u);
                for (int t = 0; t < 3; t++) fa.pool[t] = Ld.pool[t];
            }
            STAMP(13);
            fence_proxy_async();  // generic smem traffic in the ring precedes the TMA writes
            __syncthreads();
        }
        STAMP(5);

        // ================= P4: fused dequant-GEMV FFN over this CTA's share ===============
        {
            const int *loc = S.loc;
            const int cc1 = c1, cc2 = c2;
            auto src = [&](int j) -> const uint8_t * {
                const int t = j < cc1 ? 0 : (j < cc2 ? 1 : 2);
                return fa.pool[t] + (int64_t)loc[j] * fa.nb[t];
            };
            ffn_loop(fa, d, p.act, nullptr, n_items, c1, c2, src, S.ring, S.xs, S.dsc, S.bst, sm,
                     p.partial, jb, false, prof ? prof + 14 : nullptr);
            jb += (unsigned)n_items;
        }
        STAMP(6);
        grid_sync(p.bar_flags, base + ++nbar, p.err);
        STAMP(7);
        if (l == p.n_layers - 1 && cta == G - 1)  // leave both histograms clear for the next token
            for (int i = tid; i < kBins; i += NT) hist[i] = 0;

        // ================= P5: fixed-order reduction + residual ==========================
        {
            float(*rf)[33] = reinterpret_cast<float(*)[33]>(S.ring);
            for (int ch = cta; ch < d / 32; ch += G) {
                const int e = ch * 32 + lane;
                // the k_reduce order: virtual warp w sums rows w::32; two per pass, loads in flight
                for (int w = warp; w < 32; w += 2 * NW) {
                    const int w2 = w + NW;
                    float v[10], u[10];
#pragma unroll
                    for (int i = 0; i < 10; i++) {
                        const int rw = w + 32 * i, rw2 = w2 + 32 * i;
                        v[i] = rw < G ? __ldcg(p.partial + (int64_t)rw * d + e) : 0.f;
                        u[i] = (w2 < 32 && rw2 < G) ? __ldcg(p.partial + (int64_t)rw2 * d + e) : 0.f;
                    }
                    float acc = 0.f, acc2 = 0.f;
#pragma unroll
                    for (int i = 0; i < 10; i++) {
                        acc += v[i];
                        acc2 += u[i];
                    }
                    for (int rw = w + 320; rw < G; rw += 32) acc += __ldcg(p.partial + (int64_t)rw * d + e);
                    rf[w][lane] = acc;
                    if (w2 < 32) {
                        for (int rw = w2 + 320; rw < G; rw += 32) acc2 += __ldcg(p.partial + (int64_t)rw * d + e);
                        rf[w2][lane] = acc2;
                    }
                }
                __syncthreads();
                if (warp == 0) {
                    float y = 0.f;
#pragma unroll
                    for (int w = 0; w < 32; w++) y += rf[w][lane];
                    const __half yh = __float2half_rn(y);
                    p.x[e] = __hadd(__ldcg(p.x + e), yh);
                }
                __syncthreads();
            }
        }
        STAMP(8);
        if (l + 1 < p.n_layers) grid_sync(p.bar_flags, base + ++nbar, p.err);
    }
    STAMP(9);
#undef STAMP
    if (cta == 0 && tid == 0) *p.bar_epoch = base + nbar;  // the next launch is stream-ordered
}

}  // namespace

size_t decode_layer_table_bytes(int n_layers) { return sizeof(DecLayer) * (size_t)n_layers; }
size_t decode_bucket_bytes() { return (size_t)2 * kBins * kBucket * sizeof(int2); }
// scores fit the fallback buffer; a CTA's own neurons fit one pass of its threads and kOwnOff
int decode_max_F() { return (kRing - kSbufOff) / 4; }

cudaError_t init_decode_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_decode<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_decode<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    return e;
}

// host copy of the per-layer pointer table (resident layers)
cudaError_t decode_write_layer_table(m2c_ctx *c, void *dev_table) {
    std::vector<DecLayer> t(c->desc.n_layers);
    for (int l = 0; l < c->desc.n_layers; l++) {
        const LayerState &L = c->layers[l];
        t[l].A = L.A;
        t[l].B = L.B;
        for (int k = 0; k < 3; k++) t[l].pool[k] = L.pool[k];
    }
    return cudaMemcpy(dev_table, t.data(), sizeof(DecLayer) * t.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_decode(m2c_ctx *c, __half *x, unsigned long long *prof, cudaStream_t st) {
    const int d = c->desc.d_model;
    DecArgs a;
    a.layers = reinterpret_cast<const DecLayer *>(c->dec_layers);
    a.n_layers = c->desc.n_layers;
    a.d = d;
    a.r = c->desc.pred_rank;
    a.F_r = c->F_r;
    a.act = c->desc.act;
    a.k16 = c->plan.k_fp16;
    a.k8 = c->plan.k_int8;
    a.k4 = c->plan.k_int4;
    a.smax = c->sel_smax;
    a.sh = c->sel_sh;
    for (int t = 0; t < 3; t++) {
        a.nb[t] = (int)c->nb[t];
        a.wt[t] = ffn_weight(c->nb[t], d);
    }
    a.x = x;
    a.h = c->ws.h;
    a.s = c->ws.s;
    a.ghist = c->ghist;
    a.lists = c->prev_ids;
    a.partial = c->ws.partial;
    a.bar_flags = c->bar_flags;
    a.bar_epoch = c->bar_epoch;
    a.err = c->ws.err;
    a.prof = prof;
    a.bin_sh = c->dec_bin_sh;
    a.bucket = reinterpret_cast<int2 *>(c->dec_bucket);
    a.stage = c->dec_stage;
    a.ccount = c->dec_ccount;
    a.sabs = c->dec_sabs;
    // M2C_DECODE_PREFETCH: 0 none, 1 predictor slices + previous-token records (default),
    // 2 predictor slices only (tuning / measurement knob; results are identical)
    {
        const char *ev = getenv("M2C_DECODE_PREFETCH");
        a.prefetch = ev ? atoi(ev) : 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->G);
    cfg.blockDim = dim3(d / 8);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // <= 512 threads (d <= 4096): 128 registers per thread; else 64
    cudaError_t e = d / 8 <= 512 ? cudaLaunchKernelEx(&cfg, k_decode<512>, a)
                                 : cudaLaunchKernelEx(&cfg, k_decode<1024>, a);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

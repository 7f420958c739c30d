// k_decode.cu -- the persistent decode kernel: ONE cooperative launch runs a whole token
// through every layer of the resident stack (a1 -> a7 of SURVEY §8, per layer).
//
// Why: batch-1 decode of the sparse FFN moves 17.6 MB per layer at S7 (2.7 us at HBM speed)
// and 81 MB at S70H (12.4 us), while a chain of dependent kernels per layer costs ~40 us of
// launch / drain / ramp latency (round 1).  One CTA per SM stays resident for the whole token;
// the phases of a layer are separated by grid barriers (~1.3 us each on B200), THREE per
// layer:
//
//   P2  x -> smem; hq = Q(h) (h = A x was completed by integer atomics before the barrier,
//       R2); scores s = B hq of this CTA's neurons from its B slice, which the TMA engine
//       staged into shared memory during the previous layer; each score goes into a
//       4096-bin histogram (bin width 2^sh adapted per layer from the previous token's
//       max |s|) AND into that bin's bucket as a 64-bit key (s, ~id) at the slot the
//       histogram atomic returned                                                    [a2]
//   --- barrier Bs
//   P3  the selection (R3: rank order = (score desc, id asc)): every CTA copies the histogram
//       (16 KB, TMA), scans it into "keys above bin b", and derives which bins hold the ranks
//       of its own FFN share (a contiguous rank range: the shares partition the tier lists by
//       bytes + lambda x weights); it reads only those buckets, ranks their keys exactly and
//       keeps its share in rank order.  No other CTA's data is needed beyond the histogram
//       and a few buckets (round 1 copied all 148 sorted runs, 61-131 KB, into every CTA).
//       A needed bucket that overflowed (massive ties, e.g. x = 0) takes an exact block-wide
//       bisection over all scores instead.                                          [a3]
//   P4  fused dequant-GEMV FFN over the share (ffn_dev.cuh, same code as k_ffn) -> partial y
//                                                                                    [a6]
//   --- barrier By (warp 1 meanwhile stages the NEXT layer's B slice and A^T chunks into
//       shared memory by TMA)
//   R   for this CTA's 32-column chunks (concurrently, one warp group per chunk): fixed-order
//       reduction of the partial rows, x_{l+1} = fp16(x + fp16(y)) (R14); then, because
//       h = A x is exact integer arithmetic (R2), the chunk's contribution to layer l+1's h is
//       added with red.add.u64 -- order-independent, so h is bit-exact              [a7, a1]
//   --- barrier Bx (not after the last layer)
//
// Layer 0's h comes from a prologue (the R step without the reduction) and one barrier.
// Modes: whole token (resident, unsharded, or d_ff-sharded with the all-reduce fused into R
// over peer memory, §6.9); layer-split (one launch per layer, NCCL all-reduce between);
// select-only (P2 + P3 of one layer: the tier lists of the LRU/ATU engine).
// Every result is deterministic (fixed reduction orders, exact integer selection).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ffn_dev.cuh"

namespace m2c {
namespace {

constexpr int kBins = 4096;
constexpr int kCap = 128;  // bucket slots per histogram bin (more: the exact fallback)
// stamps per (layer, CTA): 0 layer start, 20 h + max, 21 hq + B slice, 22 scores, 1 P2 done, 4 after
// Bs, 2 histogram in smem, 3 scan + needed bins, 10 share ranked, 5 P3 done, 14/15 FFN
// internal (issue done / gate-up done), 6 FFN done, 7 after By, 8 R done, 9 kernel end,
// 12/13 prologue start / after its barrier
constexpr int kStamps = kDecodeStamps;
// ring offsets of the between-FFN phases (bytes)
constexpr int kRfOff = 0;          // R: partial-row sums [nc * gw][33] f32; P2: hq [r]
constexpr int kHistOff = 16384;    // P3: histogram copy [4096] i32
constexpr int kNeedOff = 49152;    // P3: needed bins / fallback candidates (16 KB)
constexpr int kAtOff = 32768;      // R: A^T chunks of the next layer (<= 32 KB, staged at By)
constexpr int kBOff = 65536;       // P2: this CTA's B slice (staged one layer ahead)
constexpr int kBMax = kRing - kBOff;

struct DecLayer {
    const int8_t *At, *B;       // A^T [d][r], B [F_r][r]
    const uint8_t *pool[3];
};

struct DecArgs {
    const DecLayer *layers;
    int n_layers, d, r, F_r, act;
    int k16, k8, k4;
    int smax;
    int nb[3], wt[3];
    __half *x;                  // [d] in/out
    long long *hb;              // [2][r][kHStride] h accumulators (layer parity)
    int *ghist;                 // [2][kBins] score histograms (layer parity)
    unsigned long long *bucket; // [2][kBins][kCap] rank keys
    int *sdump;                 // [F_r] scores of the current layer (the exact fallback)
    int32_t *lists;             // [n_layers][max(k,1)]: the selected ids in RANK order
    float *partial;             // [G][d]
    unsigned *bar_flags;        // [0] = grid-barrier arrival counter
    unsigned *bar_epoch;
    uint32_t *err;
    unsigned long long *prof;   // [n_layers][G][kStamps] globaltimer stamps, or null
    int *bin_sh;                // [n_layers] histogram scale per layer (adapted token to token)
    unsigned *sabs;             // [G] per-CTA max |s| (current layer)
    // layer-split mode (d_ff-sharded decode: one launch per layer, NCCL all-reduce between):
    const float *pre_y;         // [d] or null: the prologue first forms x = fp16(x + fp16(pre_y))
    float *post_y;              // [d] or null: R writes the reduced partial y here instead of x
    int select_only;            // 1: stop after P3 (one layer; the LRU engine follows)
    int h_ready;                // select-only: h and the histogram were prepared by the previous
                                // layer's k_reduce (no prologue, no prologue barrier)
    // §8(e) fused all-reduce over peer memory (d_ff-sharded whole-token decode):
    int nrank, rank;            // nrank > 1: the R phase exchanges the reduced y chunks
    unsigned long long *const *xpeer;  // [nrank] every rank's exchange buffer [2][nrank][d] (flag|f32)
    unsigned *rounds;           // this rank's count of completed exchanges (all layers, all tokens)
    // parity trace (m2c_set_trace, null = off): layer inputs x_l [n_layers + 1][d] fp16 and
    // the (all-reduced) layer outputs y_l [n_layers][d] f32 before rounding
    __half *xtr;
    float *ytr;
};

// histogram bin of a raw score: monotone, clamped; 2^sh-wide bins centred on 0
__device__ __forceinline__ int bin_of(int s, int sh) { return min(max((s >> sh) + 2048, 0), 4095); }
// rank key: larger key = earlier in (score desc, id asc)
__device__ __forceinline__ unsigned long long key_of(int s, int id) {
    return ((unsigned long long)((unsigned)s ^ 0x80000000u) << 32) | (unsigned)(0xffffffffu - (unsigned)id);
}
__device__ __forceinline__ int key_id(unsigned long long k) { return (int)(0xffffffffu - (unsigned)k); }

__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
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
// (wrap-safe).  ~1.3 us on B200 (round-1 microbenchmark).  Warp 1 runs `work` (latency-
// tolerant side work: TMA staging) meanwhile.  A 2 s timeout sets err bit 4 instead of hanging.
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
                flag_error(err, 4u);
                break;
            }
        }
    } else if (threadIdx.x >= 32 && threadIdx.x < 64) {
        work();
    }
    __syncthreads();
}
__device__ __forceinline__ void grid_sync(unsigned *flags, unsigned target, uint32_t *err) {
    grid_sync(flags, target, err, [] {});
}

__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v, unsigned long long *sm32) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sm32[warp] = v;
    __syncthreads();
    v = lane < nw ? sm32[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int block_sum(int v, int *sm32) {
    v = __reduce_add_sync(0xffffffffu, v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sm32[warp] = v;
    __syncthreads();
    return __reduce_add_sync(0xffffffffu, lane < nw ? sm32[lane] : 0);
}

// h_{la} += A_{la}[:, 32 ch .. 32 ch + 32) X for nc chunks at once, chunk q's fixed-point x
// values (X_j = xm_j << xsh_j, fp16_fixed) in xm[q], xsh[q]; At + q * 32 r: chunk q's 32 rows
// of A^T (global memory, or a shared-memory copy).  Two threads (adjacent lanes) per row of
// a chunk, 16 columns each, combined by one shuffle; one red.add.u64 per (chunk, row).
__device__ __forceinline__ void h_chunks(const int8_t *At, int nc, int r, const int (*xm)[32],
                                         const int (*xsh)[32], long long *hbuf) {
    for (int i2 = threadIdx.x; i2 < nc * 2 * r; i2 += blockDim.x) {  // 2 r is a multiple of 32
        const int q = i2 / (2 * r), ii = i2 - q * 2 * r;
        const int i = ii >> 1, j0 = 16 * (ii & 1);
        const int8_t *A = At + (int64_t)q * 32 * r;
        int av[16];
#pragma unroll
        for (int j = 0; j < 16; j++) av[j] = A[(int64_t)(j0 + j) * r + i];
        unsigned long long acc = 0;
#pragma unroll
        for (int j = 0; j < 16; j++) acc += (unsigned long long)(long long)(av[j] * xm[q][j0 + j]) << xsh[q][j0 + j];
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if ((ii & 1) == 0 && acc) red_add_u64(hbuf + (int64_t)i * kHStride, (long long)acc);
    }
}

template <int MAXT, bool HLDG = false>
__global__ void __launch_bounds__(MAXT, 1) k_decode(DecArgs p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    __shared__ FfnArgs fa;
    __shared__ unsigned long long red_u64[32];
    __shared__ int red_i[32];
    __shared__ int xm[2][32], xsh[2][32];
    __shared__ int nneed, ovf, share_lo, share_hi;
    __shared__ unsigned long long fb_key[2];
    __shared__ __align__(8) uint64_t sel_bar, at_bar, b_bar;
    const SmemPtrs S = carve(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5, G = gridDim.x, cta = blockIdx.x;
    const int d = p.d, r = p.r, F_r = p.F_r;
    const int kk = p.k16 + p.k8 + p.k4;
    const int nchunk = d / 32;
    const int rps = (F_r + G - 1) / G;  // neurons per CTA (this CTA: ids [n0, n1))
    const int n0 = min(F_r, cta * rps), n1 = min(F_r, n0 + rps);
    const int nown_n = n1 - n0;
    if (tid == 0) {
        ffn_init(sm, d);
        mbar_init(&sel_bar, 1);
        mbar_init(&at_bar, 1);
        mbar_init(&b_bar, 1);
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
        int lo = kk, hi = 0;
        for (int t = 0; t < 3; t++)
            if (rg[2 * t + 1] > rg[2 * t]) {
                lo = min(lo, fa.seg[t] + rg[2 * t]);
                hi = max(hi, fa.seg[t] + rg[2 * t + 1]);
            }
        if (hi <= lo) lo = hi = 0;
        share_lo = lo;  // the share is the contiguous rank range [lo, hi)
        share_hi = hi;
    }
    __syncthreads();
    const int R_lo = share_lo, R_hi = share_hi, n_items = R_hi - R_lo;
    const int c1 = min(max(p.k16 - R_lo, 0), n_items), c2 = min(max(p.k16 + p.k8 - R_lo, 0), n_items);
    // (launched with programmatic stream serialization -- select-only launches of the LRU
    // engine: the set-up above overlapped the previous kernel; nothing it wrote is read above)
    griddep_wait();
    // layer 0's B slice -> smem (arrives during the prologue)
    M2C_CHECK(nown_n * r <= kBMax && (cta < nchunk ? (nchunk - cta + G - 1) / G : 0) * 32 * r <= kBOff - kAtOff);
    if (tid == 0 && nown_n > 0) {
        mbar_expect_tx(&b_bar, (uint32_t)(nown_n * r));
        bulk_g2s_plain(S.ring + kBOff, p.layers[0].B + (int64_t)n0 * r, (uint32_t)(nown_n * r), &b_bar);
    }
    const unsigned base = ld_relaxed(p.bar_epoch);  // read by every CTA before its first arrival
    const unsigned round0 = p.nrank > 1 ? ld_relaxed(p.rounds) : 0u;
    unsigned nbar = 0;
    FfnPipe pipe;  // FFN pipeline barrier uses of this CTA so far (all layers)
    unsigned long long *prof0 = (p.prof && tid == 0) ? p.prof + (int64_t)cta * kStamps : nullptr;
    const int64_t prof_layer = (int64_t)G * kStamps;
    unsigned long long *prof = prof0;
#define STAMP(i) \
    if (prof) prof[i] = gtimer()
    STAMP(12);

    // ================= prologue: layer 0's h = A_0 x from this CTA's column chunks ==========
    for (int ch = cta; ch < nchunk && !p.h_ready; ch += G) {
        if (tid < 32) {
            bool bad = false;
            int m, sh;
            __half xv = __ldcg(p.x + ch * 32 + tid);
            if (p.pre_y) {  // the previous layer's all-reduced y (split mode): x = fp16(x + fp16(y))
                xv = __hadd(xv, __float2half_rn(__ldcg(p.pre_y + ch * 32 + tid)));
                p.x[ch * 32 + tid] = xv;
            }
            if (p.xtr) p.xtr[ch * 32 + tid] = xv;
            fp16_fixed(__half_as_ushort(xv), m, sh, bad);
            if (bad) flag_error(p.err, 1u);
            xm[0][tid] = m;
            xsh[0][tid] = sh;
        }
        __syncthreads();
        h_chunks(p.layers[0].At + (int64_t)ch * 32 * r, 1, r, xm, xsh, p.hb);
        __syncthreads();
    }
    // select-only launches leave their histogram dirty (no barrier after P3): every launch
    // clears layer 0's here, ordered before every CTA's P2 atomics by the barrier below
    if (!p.h_ready) {
        if (cta == G - 1)
            for (int i = tid; i < kBins; i += NT) p.ghist[i] = 0;
        grid_sync(p.bar_flags, base + ++nbar, p.err);
    }
    STAMP(13);

    for (int l = 0; l < p.n_layers; l++) {
        const DecLayer Ld = p.layers[l];
        int *hist = p.ghist + (l & 1) * kBins;
        unsigned long long *bkt = p.bucket + (size_t)(l & 1) * kBins * kCap;
        long long *hcur = p.hb + (int64_t)(l & 1) * r * kHStride;
        int32_t *lst = p.lists + (int64_t)l * (kk > 0 ? kk : 1);
        prof = prof0 ? prof0 + l * prof_layer : nullptr;
        STAMP(0);

        // ================= P2: x -> smem, hq = Q(h), scores, histogram + buckets ==========
        const int shl = __ldcg(p.bin_sh + l);  // this token's histogram scale for layer l
        {
            int8_t *hq = reinterpret_cast<int8_t *>(S.ring + kRfOff);
            // (h first: its L2 round trip overlaps x's instead of following it)
            long long hv0 = tid < r ? __ldcg(hcur + (int64_t)tid * kHStride) : 0;
            for (int i = tid; i < d / 8; i += NT) S.xs[i] = __ldcg(reinterpret_cast<const uint4 *>(p.x) + i);
            unsigned long long mh = (unsigned long long)(hv0 < 0 ? -hv0 : hv0);
            for (int i = tid + NT; i < r; i += NT) {
                const long long v = __ldcg(hcur + (int64_t)i * kHStride);
                mh = max(mh, (unsigned long long)(v < 0 ? -v : v));
            }
            mh = block_max_u64(mh, red_u64);
            STAMP(20);
            for (int i = tid; i < r; i += NT) {
                const long long hv = i == tid ? hv0 : __ldcg(hcur + (int64_t)i * kHStride);
                const int q = quant127_u64((unsigned long long)(hv < 0 ? -hv : hv), mh);
                hq[i] = (int8_t)(hv < 0 ? -q : q);
            }
            if (nown_n > 0) mbar_wait(&b_bar, (uint32_t)(l & 1));  // this layer's B slice
            __syncthreads();
            STAMP(21);
            // s_n = B_n . hq: LPN = min(r/16, 8) lanes per neuron, CH = r/16/LPN 16-B chunks
            // each (part + LPN c: the 8 lanes of a quarter-warp read 128 contiguous bytes of one
            // neuron, conflict-free), dp4a, shuffles over the LPN lanes -- 4 neurons per warp
            // pass at r = 256 (2 with 16 lanes of one chunk: twice the passes at S70H)
            const int LPN = min(r / 16, 8), CH = r / 16 / LPN, npw = 32 / LPN, part = lane % LPN,
                      sub = lane / LPN;
            const int4 *hq4 = reinterpret_cast<const int4 *>(hq);
            const int8_t *Bs = reinterpret_cast<const int8_t *>(S.ring + kBOff);
            int *sc = reinterpret_cast<int *>(S.ring + kHistOff);  // [nown_n] (<= 48 KB)
            for (int i0 = warp * npw; i0 < nown_n; i0 += NW * npw) {
                const int i = i0 + sub;
                int acc = 0;
                if (i < nown_n) {
#pragma unroll 4
                    for (int ch = 0; ch < CH; ch++) {
                        const int4 bv = *reinterpret_cast<const int4 *>(Bs + (int64_t)i * r + 16 * (part + LPN * ch));
                        const int4 hv4 = hq4[part + LPN * ch];
                        acc = __dp4a(bv.x, hv4.x, acc);
                        acc = __dp4a(bv.y, hv4.y, acc);
                        acc = __dp4a(bv.z, hv4.z, acc);
                        acc = __dp4a(bv.w, hv4.w, acc);
                    }
                }
                for (int o = LPN / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (part == 0 && i < nown_n) sc[i] = acc;
            }
            __syncthreads();
            STAMP(22);
            // one histogram atomic per neuron, all in flight at once; the returned slot places
            // the neuron's rank key in its bin's bucket
            unsigned smx = 0;
            for (int i = tid; i < nown_n; i += NT) {
                const int s = sc[i], n = n0 + i;
                const int b = bin_of(s, shl);
                const int pos = atomicAdd(&hist[b], 1);
                if (pos < kCap) bkt[(size_t)b * kCap + pos] = key_of(s, n);
                p.sdump[n] = s;
                smx = max(smx, (unsigned)abs(s));
            }
            smx = __reduce_max_sync(0xffffffffu, smx);
            if (lane == 0 && smx) atomicMax(&p.sabs[cta], smx);  // (reset by CTA 0 after use)
        }
        STAMP(1);
        grid_sync(p.bar_flags, base + ++nbar, p.err);
        STAMP(4);

        // ================= P3: this CTA's share of the selection, in rank order ============
        int *hs = reinterpret_cast<int *>(S.ring + kHistOff);
        int *need = reinterpret_cast<int *>(S.ring + kNeedOff);
        // HLDG (the instance for exactly 512 threads, S7): every thread loads its own run of 8
        // bins (two 16-B loads) straight into registers for the scan and keeps a copy in hs for
        // the ranking (S7 +0.8-1.2% same-box); the other instances (S70H, S13's 640 threads,
        // T's 32: 128 bins per thread) keep one TMA copy of the histogram, measured 0.6-0.9% /
        // ~10% faster there
        constexpr bool M2C_HIST_LDG = HLDG;
        if (tid == 0) {
            if (!M2C_HIST_LDG) {
                // order the ring's earlier generic accesses (and the acquired global data)
                // before the async-proxy copy
                asm volatile("fence.proxy.async;" ::: "memory");
                mbar_expect_tx(&sel_bar, (uint32_t)(4 * kBins));
                bulk_g2s_plain(hs, hist, 4 * kBins, &sel_bar);
            }
            nneed = 0;
            ovf = 0;
        }
        // per-layer bookkeeping, after Bs (every CTA's P2 is done), on three CTAs: the next
        // token's histogram scale for this layer (|s| < 2048 << sh: no clamped bins) and the
        // reset of the per-CTA max |s|; h of this layer (consumed in P2) cleared for layer
        // l+2; the other histogram (last read in layer l-1's P3) cleared for layer l+1.  It
        // runs in R on the last three CTAs when they own no R chunk (G > d/32 + 2: S7), else
        // here in P3 on the first three (their FP16-heavy FFN shares finish first: S70H)
        const bool bk_in_r = !p.select_only && G >= 3 && G - 3 >= nchunk;
        const int bk0 = bk_in_r ? G - 3 : 0;
        auto bookkeeping = [&] {
            if (cta == min(bk0, G - 1) && warp == 0) {
                unsigned m = 0;
                for (int c = lane; c < G; c += 32) m = max(m, __ldcg(p.sabs + c));
                m = __reduce_max_sync(0xffffffffu, m);
                int sh = 0;
                while ((m >> sh) >= 2048u) sh++;
                if (lane == 0) p.bin_sh[l] = sh;
                for (int c = lane; c < G; c += 32) p.sabs[c] = 0;
            }
            if (cta == min(bk0 + 1, G - 1))
                for (int i = tid; i < r; i += NT) hcur[(int64_t)i * kHStride] = 0;
            if (cta == min(bk0 + 2, G - 1))
                for (int i = tid; i < kBins; i += NT) p.ghist[((l + 1) & 1) * kBins + i] = 0;
        };
        if (!bk_in_r) bookkeeping();
        if (!M2C_HIST_LDG) mbar_wait(&sel_bar, (uint32_t)(l & 1));
        STAMP(2);
        {  // keys above each bin: per-thread runs of BPT bins (descending), block scan (warp
            // prefixes by shuffles, not a serial walk over the warps); the bins holding ranks of
            // the share go to need[] with their "above" counts at need[2048 + i]
            const int BPT = (kBins + NT - 1) / NT;  // 4 (1024 threads) .. 128 (32 threads)
            const int b_hi = max(kBins - tid * BPT, 0), b_lo = max(b_hi - BPT, 0);
            int cv[8];
            int sum = 0;
            const int *hsrc = M2C_HIST_LDG ? hist : hs;
            auto ld4 = [&](int b) {
                if (!M2C_HIST_LDG) return *reinterpret_cast<const int4 *>(hs + b);
                const int4 v = __ldcg(reinterpret_cast<const int4 *>(hist + b));
                *reinterpret_cast<int4 *>(hs + b) = v;  // (the ranking reads the counts)
                return v;
            };
            if (BPT == 8) {  // (512 threads) two 16-B loads, the run stays in registers
                const int4 v0 = ld4(b_lo);
                const int4 v1 = ld4(b_lo + 4);
                cv[0] = v1.w; cv[1] = v1.z; cv[2] = v1.y; cv[3] = v1.x;
                cv[4] = v0.w; cv[5] = v0.z; cv[6] = v0.y; cv[7] = v0.x;
                sum = (cv[0] + cv[1]) + (cv[2] + cv[3]) + ((cv[4] + cv[5]) + (cv[6] + cv[7]));
            } else if (BPT == 4) {  // (1024 threads) one 16-B load
                const int4 v0 = ld4(b_lo);
                cv[0] = v0.w; cv[1] = v0.z; cv[2] = v0.y; cv[3] = v0.x;
                sum = (cv[0] + cv[1]) + (cv[2] + cv[3]);
            } else {
                for (int b = b_hi - 1; b >= b_lo; b--) {
                    const int v = M2C_HIST_LDG ? __ldcg(hsrc + b) : hs[b];
                    if (M2C_HIST_LDG) hs[b] = v;
                    sum += v;
                }
            }
            int inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) red_i[warp] = inc;
            __syncthreads();
            int wt = lane < NW ? red_i[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, wt, o);
                if (lane >= o) wt += y;
            }
            const int wpre = warp > 0 ? __shfl_sync(0xffffffffu, wt, warp - 1) : 0;
            int acc = wpre + inc - sum;  // keys in bins >= b_hi
            auto visit = [&](int b, int c) {  // bin b (c keys), acc = keys in bins > b
                if (c > 0 && acc < R_hi && acc + c > R_lo) {  // bin b holds ranks of the share
                    const int at = atomicAdd(&nneed, 1);
                    if (at < 2048) {
                        need[at] = b;
                        need[2048 + at] = acc;
                    }
                    if (c > kCap) ovf = 1;
                }
                acc += c;
            };
            if (acc < R_hi && acc + sum > R_lo) {  // this run holds ranks of the share
                if (BPT == 8) {
#pragma unroll
                    for (int k = 0; k < 8; k++) visit(b_hi - 1 - k, cv[k]);
                } else if (BPT == 4) {
#pragma unroll
                    for (int k = 0; k < 4; k++) visit(b_hi - 1 - k, cv[k]);
                } else {
                    for (int b = b_hi - 1; b >= b_lo; b--) visit(b, hs[b]);
                }
            }
        }
        __syncthreads();
        STAMP(3);
        if (!ovf) {
            // warp per needed bin: its keys (<= kCap, 4 per lane), exact rank of each inside
            // the bin by counting larger keys; global rank = above[b] + that
            const int nn = min(nneed, 2048);
            for (int w = warp; w < nn; w += NW) {
                const int b = need[w], c = hs[b], ab = need[2048 + w];
                const unsigned long long *bk = bkt + (size_t)b * kCap;
                unsigned long long kv[4];
                int rk[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    kv[u] = lane + 32 * u < c ? __ldcg(bk + lane + 32 * u) : 0ull;
                    rk[u] = 0;
                }
                // (512 threads, d <= 4096: the specialised loops below -- S7 +0.8% same-box;
                // 1024 threads (S70H) keep the generic loop, measured 1.4% faster there)
                if (MAXT == 1024) {
#pragma unroll 1
                    for (int jj = 0; jj < c; jj++) {
                        const unsigned long long kj = __shfl_sync(0xffffffffu, kv[jj >> 5], jj & 31);
#pragma unroll
                        for (int u = 0; u < 4; u++) rk[u] += kj > kv[u];
                    }
                } else if (c <= 32) {  // (the common case: one key per lane, one compare per step)
#pragma unroll 4
                    for (int jj = 0; jj < c; jj++) rk[0] += __shfl_sync(0xffffffffu, kv[0], jj) > kv[0];
                } else {  // (static register indices: kv stays out of local memory)
#pragma unroll
                    for (int h = 0; h < 4; h++) {
                        const int m = min(32, c - 32 * h);
#pragma unroll 1
                        for (int jj = 0; jj < m; jj++) {
                            const unsigned long long kj = __shfl_sync(0xffffffffu, kv[h], jj);
#pragma unroll
                            for (int u = 0; u < 4; u++) rk[u] += kj > kv[u];
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int q = ab + rk[u];
                    if (lane + 32 * u < c && q >= R_lo && q < R_hi) {
                        const int id = key_id(kv[u]);
                        M2C_CHECK(id >= 0 && id < F_r && q < kk && q - R_lo < kMaxLocal);
                        S.loc[q - R_lo] = id;
                        lst[q] = id;
                    }
                }
            }
        } else {
            // A needed bucket overflowed (massive ties): exact block-wide bisection over all
            // scores (sdump).  key_at(q) = the key of global rank q: the largest score V with
            // #{s >= V} > q, then the (q - #{s > V})-th smallest id among s == V.
            auto count_if = [&](auto pred) {
                int c = 0;
                for (int n = tid; n < F_r; n += NT) c += pred(__ldcg(p.sdump + n), n) ? 1 : 0;
                return block_sum(c, red_i);
            };
            for (int e = 0; e < 2; e++) {
                const int q = e == 0 ? R_lo : R_hi - 1;
                int lo = -p.smax, hi = p.smax;
                while (lo < hi) {  // largest V with #{s >= V} >= q + 1
                    const int mid = lo + (hi - lo + 1) / 2;
                    if (count_if([&](int s, int) { return s >= mid; }) >= q + 1) lo = mid;
                    else hi = mid - 1;
                }
                const int V = lo;
                const int R = q - count_if([&](int s, int) { return s > V; });  // rank among s == V
                int ilo = 0, ihi = F_r - 1;
                while (ilo < ihi) {  // smallest I with #{n <= I : s_n == V} >= R + 1
                    const int mid = (ilo + ihi) >> 1;
                    if (count_if([&](int s, int n) { return s == V && n <= mid; }) >= R + 1) ihi = mid;
                    else ilo = mid + 1;
                }
                if (tid == 0) fb_key[e] = key_of(V, ilo);
                __syncthreads();
            }
            // the share = every key in [key_at(R_hi - 1), key_at(R_lo)]; rank them by counting
            const unsigned long long khi = fb_key[0], klo = fb_key[1];
            unsigned long long *cand = reinterpret_cast<unsigned long long *>(need);  // 2048 slots
            if (tid == 0) nneed = 0;
            __syncthreads();
            for (int n = tid; n < F_r; n += NT) {
                const unsigned long long kn = key_of(__ldcg(p.sdump + n), n);
                if (kn >= klo && kn <= khi) {
                    const int at = atomicAdd(&nneed, 1);
                    if (at < 2048) cand[at] = kn;
                }
            }
            __syncthreads();
            if (nneed != n_items && tid == 0) flag_error(p.err, 8u);
            const int m = min(nneed, n_items);
            for (int i = tid; i < m; i += NT) {
                int rk = 0;
                for (int j = 0; j < m; j++) rk += cand[j] > cand[i];
                const int id = key_id(cand[i]);
                M2C_CHECK(id >= 0 && id < F_r && rk < n_items);
                S.loc[rk] = id;
                lst[R_lo + rk] = id;
            }
        }
        STAMP(10);
        if (tid == 0)
            for (int t = 0; t < 3; t++) fa.pool[t] = Ld.pool[t];
        fence_proxy_async();  // generic smem traffic in the ring precedes the FFN's TMA writes
        __syncthreads();
        STAMP(5);
        if (p.select_only) break;  // the LRU/ATU engine: the lists are out (the histogram is
                                    // cleared by the next launch's prologue)

        // ================= P4: fused dequant-GEMV FFN over this CTA's share ===============
        {
            const int *loc = S.loc;
            auto src = [&](int j) -> const uint8_t * {
                const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
                M2C_CHECK(j >= 0 && j < n_items && loc[j] >= 0 && loc[j] < F_r);
                return fa.pool[t] + (int64_t)loc[j] * fa.nb[t];
            };
            ffn_run(fa, d, p.act, n_items, c1, c2, src, S.ring, S.xs, S.a, sm, pipe, p.partial,
                    prof ? prof + 14 : nullptr);
        }
        STAMP(6);
        // barrier By; meanwhile (warp 1): layer l+1's A^T chunks of this CTA (for R) and its
        // B slice (for P2) -> smem by TMA
        const bool more = l + 1 < p.n_layers;
        const int nown_c = cta < nchunk ? (nchunk - cta + G - 1) / G : 0;
        grid_sync(p.bar_flags, base + ++nbar, p.err, [&] {
            if (more && (threadIdx.x & 31) == 0) {
                fence_proxy_async();  // the FFN's generic reads of the ring precede the copies
                if (nown_c > 0) {
                    const uint32_t bytes = 32u * (uint32_t)r;
                    mbar_expect_tx(&at_bar, bytes * nown_c);
                    for (int q = 0; q < nown_c; q++)
                        bulk_g2s_plain(S.ring + kAtOff + q * bytes,
                                       p.layers[l + 1].At + (int64_t)(cta + q * G) * bytes, bytes, &at_bar);
                }
                if (nown_n > 0) {
                    mbar_expect_tx(&b_bar, (uint32_t)(nown_n * r));
                    bulk_g2s_plain(S.ring + kBOff, p.layers[l + 1].B + (int64_t)n0 * r,
                                   (uint32_t)(nown_n * r), &b_bar);
                }
            }
        });
        STAMP(7);
        // (each layer's histogram is cleared by the previous layer's bookkeeping, layer 0's by
        // the prologue)

        // ================= R: fixed-order reduction + residual + next layer's h ==============
        {
            long long *hnext = p.hb + (int64_t)((l + 1) & 1) * r * kHStride;
            const __half *xs_h = reinterpret_cast<const __half *>(S.xs);
            const int P = p.nrank;
            const unsigned flag = round0 + (unsigned)l + 1u;
            const size_t row = (size_t)((flag - 1u) & 1u) * P;
            const int ncc = min(nown_c, min(2, NW));  // chunks reduced concurrently
            if (more && nown_c > 0) mbar_wait(&at_bar, (uint32_t)(l & 1));  // A^T chunks staged at By
            for (int q0 = 0; q0 < nown_c; q0 += ncc) {
                const int nc = min(ncc, nown_c - q0);
                const int gw = NW / nc;  // warps per chunk
                float(*rf)[33] = reinterpret_cast<float(*)[33]>(S.ring + kRfOff);  // [nc * gw][33]
                const int g = warp / gw, v = warp - g * gw;
                const int e = (cta + (q0 + g) * G) * 32 + lane;
                if (g < nc) {  // group g reduces chunk q0 + g: virtual warp v sums rows v::gw,
                    // up to 12 rows' loads in flight before the (fixed-order) sum
                    float acc = 0.f;
                    for (int rw0 = v; rw0 < G; rw0 += 12 * gw) {
                        float pv[12];
#pragma unroll
                        for (int i = 0; i < 12; i++) {
                            const int rw = rw0 + i * gw;
                            pv[i] = rw < G ? __ldcg(p.partial + (int64_t)rw * d + e) : 0.f;
                        }
#pragma unroll
                        for (int i = 0; i < 12; i++) acc += pv[i];
                    }
                    rf[g * gw + v][lane] = acc;
                }
                __syncthreads();
                if (g < nc && v == 0) {  // the group's first warp: y of its chunk
                    float y = 0.f;
                    for (int w = 0; w < gw; w++) y += rf[g * gw + w][lane];
                    if (P > 1) {
                        // the all-reduce fused into the reduction (§6.9): this rank's y of the
                        // element goes into every rank's exchange buffer as a (flag | value)
                        // 8-byte word (peer stores over NVLink; complete when its flag matches --
                        // no fences, no counters), then the P words of this rank's buffer are
                        // summed in rank order
                        const unsigned long long wv = ((unsigned long long)flag << 32) | __float_as_uint(y);
                        for (int qq = 0; qq < P; qq++) st_relaxed_sys_u64(p.xpeer[qq] + (row + p.rank) * d + e, wv);
                        const unsigned long long *mine = p.xpeer[p.rank] + row * d + e;
                        y = 0.f;
                        for (int qq = 0; qq < P; qq++) {
                            unsigned long long w = ld_relaxed_sys_u64(mine + (size_t)qq * d);
                            if ((unsigned)(w >> 32) != flag &&
                                !(*reinterpret_cast<volatile unsigned *>(p.err) & 16u)) {
                                // (after one timeout no CTA waits again: a dead peer costs 5 s
                                // per token, not per chunk)
                                const unsigned long long t0 = gtimer();
                                do {
                                    w = ld_relaxed_sys_u64(mine + (size_t)qq * d);
                                    if (gtimer() - t0 > 5000000000ull) {
                                        flag_error(p.err, 16u);
                                        break;
                                    }
                                } while ((unsigned)(w >> 32) != flag);
                            }
                            y += __uint_as_float((unsigned)w);
                        }
                    }
                    const __half xn = __hadd(xs_h[e], __float2half_rn(y));
                    if (p.post_y) {
                        p.post_y[e] = y;  // split mode: this rank's y, to be all-reduced
                    } else {
                        p.x[e] = xn;
                        if (p.ytr) p.ytr[(int64_t)l * d + e] = y;
                        if (p.xtr) p.xtr[(int64_t)(l + 1) * d + e] = xn;
                    }
                    if (more) {
                        bool bad = false;
                        int m, sh;
                        fp16_fixed(__half_as_ushort(xn), m, sh, bad);
                        if (bad) flag_error(p.err, 1u);
                        xm[g][lane] = m;
                        xsh[g][lane] = sh;
                    }
                }
                __syncthreads();
                if (more) {
                    h_chunks(reinterpret_cast<const int8_t *>(S.ring + kAtOff) + (int64_t)q0 * 32 * r, nc, r,
                             xm, xsh, hnext);
                    __syncthreads();
                }
            }
        }
        if (bk_in_r) bookkeeping();
        STAMP(8);
        if (more) grid_sync(p.bar_flags, base + ++nbar, p.err);
    }
    STAMP(9);
#undef STAMP
    if (cta == 0 && tid == 0) {
        *p.bar_epoch = base + nbar;  // the next launch is stream-ordered
        if (p.nrank > 1) *p.rounds = round0 + (unsigned)p.n_layers;
    }
}

// ---- tier lists in rank order -> three ascending-id segments (select-only output and
// m2c_decode_lists): one CTA per tier.  The ids are distinct integers in [0, F_r): each sets its
// bit in a shared-memory bitmap, a block scan of the words' popcounts gives every word's output
// position, and each thread writes its word's ids in ascending order (O(F_r / 32 + n), three
// barriers; the round-1 bitonic network took ~55 barriers, 11.7 us per layer at S13).
__global__ void __launch_bounds__(1024) k_sort_tiers(int32_t *ids, int seg1, int seg2, int n0, int n1,
                                                     int n2, int F_r) {
    extern __shared__ __align__(16) uint32_t bm[];  // [ceil(F_r / 32)] bitmap | [32] warp sums
    griddep_wait();
    const int t = blockIdx.x;
    const int seg = t == 0 ? 0 : (t == 1 ? seg1 : seg2), n = t == 0 ? n0 : (t == 1 ? n1 : n2);
    if (n <= 1) return;
    const int W = (F_r + 31) >> 5, NT = blockDim.x;
    int *wsum = reinterpret_cast<int *>(bm + W);
    for (int w = threadIdx.x; w < W; w += NT) bm[w] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) {
        const int id = ids[seg + i];
        atomicOr(&bm[id >> 5], 1u << (id & 31));
    }
    __syncthreads();
    // each thread owns the words [w0, w1) (contiguous), block exclusive scan of their popcounts
    const int per = (W + NT - 1) / NT;
    const int w0 = min(W, (int)threadIdx.x * per), w1 = min(W, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; w++) cnt += __popc(bm[w]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int wt = lane < (NT >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wt, o);
        if (lane >= o) wt += y;
    }
    int pos = (warp > 0 ? __shfl_sync(0xffffffffu, wt, warp - 1) : 0) + inc - cnt;
    for (int w = w0; w < w1; w++) {
        uint32_t b = bm[w];
        while (b) {
            const int k = __ffs(b) - 1;
            b &= b - 1;
            ids[seg + pos++] = (w << 5) + k;
        }
    }
}
constexpr int kSortMax = 32768;   // entries per tier (m2c_decode_lists' limit)
constexpr int kSortFr = 1 << 20;  // F_r covered by k_sort_tiers' bitmap (128 KB of smem)

}  // namespace

size_t decode_layer_table_bytes(int n_layers) { return sizeof(DecLayer) * (size_t)n_layers; }
size_t decode_hist_bytes() { return sizeof(int) * 2 * (size_t)kBins; }
size_t decode_bucket_bytes() { return sizeof(unsigned long long) * 2 * (size_t)kBins * kCap; }
int sort_tiers_max() { return kSortMax; }
// the shapes k_decode covers: this CTA's B slice fits the ring's B region and the largest
// FFN share fits kMaxLocal (r <= 512 and d <= 8192 by check_desc)
bool decode_shape_ok(const m2c_ctx *c) {
    const int G = c->G;
    const int64_t rps = (c->F_r + G - 1) / G;
    if (rps * c->desc.pred_rank > kBMax || rps > 12288) return false;  // B slice, scores scratch
    const int d = c->desc.d_model;
    const int64_t w[3] = {ffn_weight(c->nb[0], d), ffn_weight(c->nb[1], d), ffn_weight(c->nb[2], d)};
    const int64_t W = c->plan.k_fp16 * w[0] + c->plan.k_int8 * w[1] + c->plan.k_int4 * w[2];
    const int64_t wmin = std::min(w[0], std::min(w[1], w[2]));
    return W / G / wmin + 4 <= kMaxLocal;
}

cudaError_t init_decode_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_decode<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_decode<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_decode<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_sort_tiers, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * (kSortFr / 32 + 32));
    return e;
}

cudaError_t launch_sort_tiers(m2c_ctx *c, int32_t *ids, const m2c_tier_plan &p, cudaStream_t st) {
    if (c->F_r > kSortFr) return cudaErrorInvalidValue;
    const size_t smem = 4 * ((size_t)(c->F_r + 31) / 32 + 32);
    cudaError_t e = launch_k(k_sort_tiers, dim3(3), dim3(1024), smem, st, ids, p.k_fp16, p.k_fp16 + p.k_int8,
                             p.k_fp16, p.k_int8, p.k_int4, c->F_r);
    c->launch_counter++;
    return e;
}

// host copy of the per-layer pointer table (resident layers)
cudaError_t decode_write_layer_table(m2c_ctx *c, void *dev_table) {
    std::vector<DecLayer> t(c->desc.n_layers);
    for (int l = 0; l < c->desc.n_layers; l++) {
        const LayerState &L = c->layers[l];
        t[l].At = L.A;
        t[l].B = L.B;
        for (int k = 0; k < 3; k++) t[l].pool[k] = L.pool[k];
    }
    return cudaMemcpy(dev_table, t.data(), sizeof(DecLayer) * t.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_decode(m2c_ctx *c, __half *x, unsigned long long *prof, cudaStream_t st, int layer0,
                          int nl, const float *pre_y, float *post_y, int32_t *lists_out, bool h_ready) {
    const int d = c->desc.d_model;
    if (nl < 0) nl = c->desc.n_layers - layer0;
    DecArgs a;
    a.layers = reinterpret_cast<const DecLayer *>(c->dec_layers) + layer0;
    a.n_layers = nl;
    a.pre_y = pre_y;
    a.post_y = post_y;
    a.d = d;
    a.r = c->desc.pred_rank;
    a.F_r = c->F_r;
    a.act = c->desc.act;
    a.k16 = c->plan.k_fp16;
    a.k8 = c->plan.k_int8;
    a.k4 = c->plan.k_int4;
    a.smax = c->sel_smax;
    for (int t = 0; t < 3; t++) {
        a.nb[t] = (int)c->nb[t];
        a.wt[t] = ffn_weight(c->nb[t], d);
    }
    a.x = x;
    a.hb = c->dec_hb;
    a.ghist = c->dec_hist;
    a.bucket = c->dec_bucket;
    a.sdump = c->dec_sdump;
    a.lists = lists_out ? lists_out : c->prev_ids + (size_t)layer0 * (c->plan.k > 0 ? c->plan.k : 1);
    a.select_only = lists_out != nullptr;
    a.h_ready = (lists_out && h_ready) ? 1 : 0;
    a.nrank = (c->p2p && !lists_out && !post_y) ? c->desc.shard_count : 1;
    a.rank = c->desc.shard_index;
    a.xpeer = c->p2p_xtab;
    a.rounds = c->p2p_rounds;
    a.partial = c->ws.partial;
    a.bar_flags = c->bar_flags;
    a.bar_epoch = c->bar_epoch;
    a.err = c->ws.err;
    a.prof = prof ? prof + (size_t)layer0 * c->G * kStamps : nullptr;
    a.bin_sh = c->dec_bin_sh + layer0;
    a.sabs = c->dec_sabs;
    a.xtr = (c->trace_x && !lists_out) ? c->trace_x + (size_t)layer0 * d : nullptr;
    a.ytr = (c->trace_y && !lists_out && !post_y) ? c->trace_y + (size_t)layer0 * d : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->G);
    cfg.blockDim = dim3(d / 8);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (lists_out) {  // select-only (LRU engine): overlap the launch with the previous kernel
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs = 2;
    }
    // <= 512 threads (d <= 4096): 128 registers per thread; else 64 (exactly 512: the instance
    // with the register-run histogram load)
    cudaError_t e = d / 8 == 512  ? cudaLaunchKernelEx(&cfg, k_decode<512, true>, a)
                    : d / 8 < 512 ? cudaLaunchKernelEx(&cfg, k_decode<512>, a)
                                  : cudaLaunchKernelEx(&cfg, k_decode<1024>, a);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

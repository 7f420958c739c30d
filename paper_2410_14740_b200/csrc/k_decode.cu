// k_decode.cu -- the persistent decode kernel: ONE cooperative launch runs a whole token
// through every layer of the resident stack (a1 -> a7 of SURVEY §8, per layer).
//
// Why: batch-1 decode of the sparse FFN moves ~17 MB per layer (S7), i.e. ~2.7 us at HBM
// speed, while a chain of dependent kernels per layer costs ~40 us of launch / drain / ramp
// latency (profiles/).  One CTA per SM stays resident for the whole token; the phases of a
// layer are separated by grid barriers (~1.3 us each on B200, tools/mb_gridsync2.cu), so the
// design minimises their number: THREE per layer.
//
//   P2  hq = Q(h) (every CTA: h = A x was completed by integer atomics before the barrier),
//       x -> smem, scores s = B hq of this CTA's neurons, 4096-bin score histogram (global
//       atomics)                                                                     [a2]
//   --- barrier Bs
//   P3  every CTA pulls the whole histogram and ALL scores into shared memory with two TMA
//       bulk copies and derives the selection itself: the three rank cuts (k16, k16+k8, k;
//       histogram scans, exact ranking of the cut bins' candidates, ties by id -- R3), then a
//       block-wide ordered compaction that keeps the ids falling into this CTA's share of the
//       tier lists.  No exchange is needed: the lists are a pure function of s.         [a3]
//   P4  fused dequant-GEMV FFN over the share (ffn_dev.cuh, same code as k_ffn) -> partial y
//                                                                                    [a6]
//   --- barrier By
//   R   for this CTA's 32-column chunks: fixed-order reduction of the partials (the k_reduce
//       order), x_{l+1} = fp16(x + fp16(y)) (R14); then, because h = A x is exact integer
//       arithmetic (R2), the chunk's contribution to layer l+1's h = A_{l+1} x_{l+1} is added
//       with red.add.u64 -- integer atomics are order-independent, so h is bit-exact and the
//       predictor needs no barrier of its own                                     [a7, a1]
//   --- barrier Bx (not after the last layer)
//
// Layer 0's h comes from a prologue (the R step without the reduction) and one barrier.
// At barrier By, warp 1 stages this CTA's A^T chunk of layer l+1 into shared memory (TMA) for
// R.  An optional L2 lookahead (M2C_DECODE_PREFETCH) streams layer l+1's predictor slice and
// the records the previous token selected for layer l+1 (~80% recur); it is off by
// default: the FFN's own reads already run at HBM speed (~1.8 us for 13.75 MB at S7) and the
// prefetch traffic slows the latency-bound phases more than it saves (tools/exp_prefetch.sh).
// Results are bit-identical to the per-phase kernel chain (same select rule, same per-CTA FFN
// shares and batches, same reduction order): tests/test_gpu_parity.py checks it.
#include <cstdlib>

#include "ffn_dev.cuh"

namespace m2c {
namespace {

#ifndef M2C_CAND_WALK
#define M2C_CAND_WALK 1  // candidates: one binary search + a walk over the bin's members (A/B: 662 vs 676 us)
#endif
#ifndef M2C_BAR_MODE
#define M2C_BAR_MODE 1
#endif
constexpr int kBins = 4096;
constexpr int kHistW = kBins + 64;  // fine bins, then 64 coarse bins (CTA-aggregated atomics)
// profiling stamps per (layer, CTA): 0 layer start, 1 P2 done, 4 after Bs, 2 runs in smem,
// 3 cut bins found, 10 cuts exact,
// 11 lists done, 5 P3 done, 6 P4 done, 7 after By, 8 R done, 9 kernel end (last layer),
// 12/13 prologue start / after its barrier (layer 0), 14/15 FFN-internal (ffn_loop)
constexpr int kStamps = kDecodeStamps;
constexpr int kCand = 64;         // candidates ranked per cut bin (more: block-wide fallback)
// ring-aliased scratch of P2..P3 (bytes): hq [0, 512) | histogram + coarse sums [4K, 20.25K)
// | cut candidates [21K, 22.5K) | all scores from 32K
constexpr int kHistOff = 4096;
constexpr int kCandOff = 21504;
constexpr int kCcOff = 23040;     // [G][4] per-run cumulative tier counts (G <= 148)
constexpr int kExOff = 25600;     // [G][4] per-run list positions (before: per-run cut keys)
constexpr int kWorkOff = 28160;   // [<= 3 G] (run, tier) work items of the list write
constexpr int kSbufOff = 32768;
// R: this CTA's A^T chunks of the next layer (<= 2 x 32 r bytes), staged by TMA at barrier By
constexpr int kAtOff = 8192;

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
    int *runs;                  // [G][RP] per-CTA sorted score keys (P2 -> P3)
    int *ghist;                 // [2][kHistW] fine + coarse score histograms (layer parity)
    int T;                      // run row length (== RP)
    int32_t *lists;             // [n_layers][max(k,1)]  (the tier lists; next token's prefetch hint)
    float *partial;             // [G][d]
    unsigned *bar_flags;        // [0] = grid-barrier arrival counter
    unsigned *bar_epoch;
    uint32_t *err;
    unsigned long long *prof;   // [n_layers][G][kStamps] globaltimer stamps, or null
    int prefetch;
    int *bin_sh;                // [n_layers] histogram scale per layer (adapted token to token)
    unsigned *sabs;             // [2G] per-CTA |s| of its run's two ends (current layer)
    // layer-split mode (d_ff-sharded decode: one launch per layer, NCCL all-reduce between):
    const float *pre_y;         // [d] or null: the prologue first forms x = fp16(x + fp16(pre_y))
    float *post_y;              // [d] or null: R writes the reduced partial y here instead of x
    int select_only;            // 1: stop after P3 (one layer; the chain's cache + FFN follow)
    // §8(e) fused all-reduce over peer memory (d_ff-sharded whole-token decode):
    int nrank, rank;            // nrank > 1: the R phase exchanges the reduced y chunks
    unsigned long long *const *xpeer;  // [nrank] every rank's exchange buffer [2][nrank][d] (flag|f32)
    unsigned *rounds;           // this rank's count of completed exchanges (all layers, all tokens)
};

// histogram bin of a raw score: monotone, clamped; 2^sh-wide bins centred on 0
__device__ __forceinline__ int bin_of(int s, int sh) { return min(max((s >> sh) + 2048, 0), 4095); }

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
// (wrap-safe).  Measured ~1.3 us on B200 (tools/mb_gridsync2.cu).  Warp 1 runs `work`
// (latency-tolerant side work) meanwhile.  A 2 s timeout sets err bit 4 instead of hanging.
template <class F>
__device__ __forceinline__ void grid_sync(unsigned *counter, unsigned target, uint32_t *err, F work) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockDim.x == 32) work();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
        const unsigned want = target * gridDim.x;
        const unsigned long long t0 = gtimer();
#if M2C_BAR_MODE == 2  // relaxed polling, one acquire fence after
        while ((int)(ld_relaxed(counter) - want) < 0) {
#else
        while ((int)(ld_acquire(counter) - want) < 0) {
#endif
            if (gtimer() - t0 > 2000000000ull) {
                flag_error(err, 4u);
                break;
            }
        }
#if M2C_BAR_MODE == 2
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
    } else if (threadIdx.x >= 32 && threadIdx.x < 64) {
        work();  // warp 1: e.g. L2 prefetch while thread 0 waits
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
// one L2 prefetch of [p, p + bytes): a TMA bulk prefetch (mode 1, 2), or per-line
// prefetch.global.L2 instructions spread over the warp (mode 3, 4: LSU path, no TMA queue)
__device__ __forceinline__ void pf_range(int mode, const void *ptr, uint32_t bytes, int lane, int nl) {
    if (mode <= 2) {
        if (lane == 0) prefetch_l2(ptr, bytes);
    } else {
        const char *c = static_cast<const char *>(ptr);
        for (uint32_t o = 128u * lane; o < bytes; o += 128u * nl)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
    }
}

// L2 prefetch (one warp, fire and forget): this CTA's predictor slice of layer lb (B rows of
// its neurons), its A^T chunks of layer la, its share of the records the previous token
// selected for layer lr.  Negative layer indices skip that part.
// M2C_DECODE_PREFETCH: 0 none; 1 all (TMA bulk prefetch); 2 predictor only (TMA);
// 3 all (per-line LSU prefetch); 4 predictor only (LSU).
__device__ __forceinline__ void prefetch_layers(const DecArgs &p, int lb, int la, int lr) {
    const int mode = p.prefetch;
    if (mode == 0) return;
    const int lane = threadIdx.x & 31, G = gridDim.x, cta = blockIdx.x;
    const int nl = blockDim.x == 32 ? 1 : 32;  // a 32-thread CTA runs this on thread 0 alone
    const int ln = blockDim.x == 32 ? 0 : lane;
    if (lb >= 0) {
        const int8_t *B = p.layers[lb].B;
        const int rps = (p.F_r + G - 1) / G;
        const int n0 = cta * rps, n1 = min(p.F_r, n0 + rps);
        if (n1 > n0) pf_range(mode, B + (int64_t)n0 * p.r, (uint32_t)((n1 - n0) * p.r), ln, nl);
    }
    if (la >= 0) {
        const int8_t *At = p.layers[la].At;
        for (int ch = cta; ch < p.d / 32; ch += G) pf_range(mode, At + (int64_t)ch * 32 * p.r, (uint32_t)(32 * p.r), ln, nl);
    }
    if (lr >= 0 && (mode == 1 || mode == 3)) {
        const DecLayer Lj = p.layers[lr];
        const int k = p.k16 + p.k8 + p.k4;
        const int32_t *ids = p.lists + (int64_t)lr * (k > 0 ? k : 1);
        const int i0 = (int)((long long)k * cta / G), i1 = (int)((long long)k * (cta + 1) / G);
        if (mode == 1) {
            for (int i = i0 + ln; i < i1; i += nl) {
                const int t = i < p.k16 ? 0 : (i < p.k16 + p.k8 ? 1 : 2);
                const int id = __ldcg(ids + i);
                if (id >= 0 && id < p.F_r) prefetch_l2(Lj.pool[t] + (int64_t)id * p.nb[t], (uint32_t)p.nb[t]);
            }
        } else {
            for (int i = i0; i < i1; i++) {
                const int t = i < p.k16 ? 0 : (i < p.k16 + p.k8 ? 1 : 2);
                const int id = __ldcg(ids + i);
                if (id >= 0 && id < p.F_r) pf_range(mode, Lj.pool[t] + (int64_t)id * p.nb[t], (uint32_t)p.nb[t], ln, nl);
            }
        }
    }
}

// h_{la} += A_{la}[:, 32 ch .. 32 ch + 32) X for the chunk whose fixed-point x values
// (X_j = xm_j << xsh_j, fp16_fixed) are in shared memory; one red.add.u64 per row.
// At: the chunk's 32 rows of A^T (global memory, or a shared-memory copy)
// Two threads (adjacent lanes) per row, 16 columns each, combined by one shuffle.
__device__ __forceinline__ void h_chunk(const int8_t *At, int r, const int *xm, const int *xsh,
                                        long long *hbuf) {
    for (int i2 = threadIdx.x; i2 < 2 * r; i2 += blockDim.x) {  // 2 r is a multiple of 32
        const int i = i2 >> 1, j0 = 16 * (i2 & 1);
        int av[16];
#pragma unroll
        for (int j = 0; j < 16; j++) av[j] = At[(int64_t)(j0 + j) * r + i];
        unsigned long long acc = 0;
#pragma unroll
        for (int j = 0; j < 16; j++) acc += (unsigned long long)(long long)(av[j] * xm[j0 + j]) << xsh[j0 + j];
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if ((i2 & 1) == 0 && acc) red_add_u64(hbuf + (int64_t)i * kHStride, (long long)acc);
    }
}

template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_decode(DecArgs p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    __shared__ FfnArgs fa;
    __shared__ unsigned long long red_u64[32];
    __shared__ int red_i[32];
    __shared__ int cut_bin[3], cut_need[3], cut_V[3], cut_I[3], ncand[3], ccnt[3];
    __shared__ int xm[32], xsh[32];
    __shared__ int ccoarse[64];
    __shared__ __align__(8) uint64_t sel_bar, at_bar;
    const SmemPtrs S = carve(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5, G = gridDim.x, cta = blockIdx.x;
    const int d = p.d, r = p.r, F_r = p.F_r;
    const int kk = p.k16 + p.k8 + p.k4;
    auto tg = [&](int t) { return t == 0 ? p.k16 : (t == 1 ? p.k16 + p.k8 : kk); };  // cut targets
    const int nchunk = d / 32;
    if (tid == 0) {
        ffn_init_bars(sm);
        mbar_init(&sel_bar, 1);
        mbar_init(&at_bar, 1);
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
    // (launched with programmatic stream serialization -- select-only launches of the LRU chain:
    // the set-up above overlapped the previous kernel; nothing it wrote is read before here)
    griddep_wait();
    const unsigned base = ld_relaxed(p.bar_epoch);  // read by every CTA before its first arrival
    const unsigned round0 = p.nrank > 1 ? ld_relaxed(p.rounds) : 0u;
    unsigned nbar = 0;
    unsigned jb = 0;  // mbarrier uses of this CTA so far
    // per-CTA globaltimer stamps (profiling): [l][cta][kStamps], see STAMP below
    unsigned long long *prof0 = (p.prof && tid == 0) ? p.prof + (int64_t)cta * kStamps : nullptr;
    const int64_t prof_layer = (int64_t)G * kStamps;
    unsigned long long *prof = prof0;
#define STAMP(i) \
    if (prof) prof[i] = gtimer()
    STAMP(12);
    if (warp == NW - 1) prefetch_layers(p, 0, p.n_layers > 1 ? 1 : -1, 0);
    // (the L2 prefetches are bulk operations of the SM's TMA unit, which serves requests in
    // order: they are issued where no latency-critical copy is queued behind them -- here and
    // at barrier By, after the FFN's copies)

    // ================= prologue: layer 0's h = A_0 x from this CTA's column chunks ==========
    for (int ch = cta; ch < nchunk; ch += G) {
        if (tid < 32) {
            bool bad = false;
            int m, sh;
            __half xv = __ldcg(p.x + ch * 32 + tid);
            if (p.pre_y) {  // the previous layer's all-reduced y (split mode): x = fp16(x + fp16(y))
                xv = __hadd(xv, __float2half_rn(__ldcg(p.pre_y + ch * 32 + tid)));
                p.x[ch * 32 + tid] = xv;
            }
            fp16_fixed(__half_as_ushort(xv), m, sh, bad);
            if (bad) flag_error(p.err, 1u);
            xm[tid] = m;
            xsh[tid] = sh;
        }
        __syncthreads();
        h_chunk(p.layers[0].At + (int64_t)ch * 32 * r, r, xm, xsh, p.hb);
        __syncthreads();
    }
    // select-only launches leave their histogram dirty (no barrier after P3): every launch
    // clears layer 0's here, ordered before every CTA's P2 atomics by the barrier below
    if (cta == G - 1)
        for (int i = tid; i < kHistW; i += NT) p.ghist[i] = 0;
    grid_sync(p.bar_flags, base + ++nbar, p.err);
    STAMP(13);

    for (int l = 0; l < p.n_layers; l++) {
        const DecLayer Ld = p.layers[l];
        int *hist = p.ghist + (l & 1) * kHistW;
        long long *hcur = p.hb + (int64_t)(l & 1) * r * kHStride;
        int32_t *lst = p.lists + (int64_t)l * (kk > 0 ? kk : 1);
        prof = prof0 ? prof0 + l * prof_layer : nullptr;
        STAMP(0);

        // ================= P2: hq = Q(h), x -> smem, scores, histogram, sorted run ==========
        for (int i = tid; i < 64; i += NT) ccoarse[i] = 0;  // (published after the scores' barrier below)
        const int shl = __ldcg(p.bin_sh + l);  // this token's histogram scale for layer l
        const int rps = (F_r + G - 1) / G;      // neurons per CTA (this CTA: ids [n0, n1))
        const int RP = rps | 1;  // run row length: odd, so same-index probes of 32 runs hit 32 banks
        {
            int8_t *hq = reinterpret_cast<int8_t *>(S.ring);
            int *keys = reinterpret_cast<int *>(S.ring + 1024);  // this CTA's run keys (<= 256)
            // lanes per neuron LPN, 16-B chunks per lane CPL (r = 256: 4 x 4; r = 32: 1 x 2)
            const int C16 = r / 16, CPL = C16 >= 4 ? 4 : C16, LPN = C16 / CPL, npw = 32 / LPN;
            const int part = lane % LPN, sub = lane / LPN;
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
            S.xs[tid] = __ldcg(reinterpret_cast<const uint4 *>(p.x) + tid);  // NT == d / 8
            long long hv0 = tid < r ? __ldcg(hcur + (int64_t)tid * kHStride) : 0;
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
            __syncthreads();
            STAMP(21);
            const int4 *hq4 = reinterpret_cast<const int4 *>(hq) + part * CPL;
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
                    // run key: (s, local index asc) in one int -- |s| < 2^23 (R2), local < 255
                    keys[n - n0] = (int)(((unsigned)acc << 8) | (unsigned)(255 - (n - n0)));
                    const int b = bin_of(acc, shl);
                    atomicAdd(&hist[b], 1);
                    atomicAdd(&ccoarse[b >> 6], 1);  // smem: this CTA's coarse counts
                }
                nb0 += step;
                if (nb0 < n1) load_b();
            }
            STAMP(22);
            __syncthreads();  // keys[] and the coarse counts complete
            for (int i = tid; i < 64; i += NT)
                if (ccoarse[i]) atomicAdd(&hist[kBins + i], ccoarse[i]);
            // sorted run (key descending): rank by counting, four threads per key (a quarter of
            // the comparisons each, combined by shuffles within the aligned group of four)
            const int nown = n1 - n0;
            int *run = p.runs + (int64_t)cta * RP;
            for (int i4 = tid; i4 < ((4 * RP + 31) & ~31); i4 += NT) {  // whole warps (shuffles)
                const int i = i4 >> 2, part4 = i4 & 3;
                const int ki = i < nown ? keys[i] : (int)0x80000000;
                int rk = 0;
                for (int j = part4; j < nown; j += 4) rk += keys[j] > ki;
                rk += __shfl_xor_sync(0xffffffffu, rk, 1);
                rk += __shfl_xor_sync(0xffffffffu, rk, 2);
                if (part4 == 0 && i < RP) run[i < nown ? rk : i] = ki;  // padding keeps its slot
                // max |s| of this CTA (next token's histogram scale): the run's two ends
                if (part4 == 0 && i < nown && (rk == 0 || rk == nown - 1))
                    p.sabs[2 * cta + (rk != 0)] = (unsigned)abs(ki >> 8);
            }
        }
        STAMP(1);
        grid_sync(p.bar_flags, base + ++nbar, p.err);
        STAMP(4);

        // ================= P3: the selection, every CTA from a copy of all sorted runs =========
        int *hs = reinterpret_cast<int *>(S.ring + kHistOff);
        const int T = p.T;
        const int *ts = reinterpret_cast<const int *>(S.ring + kSbufOff);  // all runs [G][RP]
        // key e of run c: the smem copy of the run's first T keys, else the run in global memory
        auto runkey = [&](int c, int e) { return ts[c * T + e]; };  // T == RP: every run is in smem
        if (tid == 0) {  // histograms + run prefixes -> smem: two bulk copies on one mbarrier
            // order the ring's earlier generic accesses (and the acquired global data) before
            // the async-proxy copies
            asm volatile("fence.proxy.async;" ::: "memory");
            const uint32_t sb = (uint32_t)((4 * G * T + 15) & ~15);  // (the buffer has slack)
            mbar_expect_tx(&sel_bar, (uint32_t)(4 * kHistW) + sb);
            bulk_g2s_plain(hs, hist, 4 * kHistW, &sel_bar);
            bulk_g2s_plain(S.ring + kSbufOff, p.runs, sb, &sel_bar);
        }
        if (tid < 3) {
            cut_V[tid] = 0x7fffffff;  // empty cut: nothing is above it
            cut_I[tid] = -1;
            cut_bin[tid] = -1;
            ncand[tid] = 0;
            ccnt[tid] = 0;
        }
        // next token's histogram scale for this layer: |s| < 2048 << sh (no clamped bins)
        if (cta == 0 && warp == 0) {
            unsigned m = 0;
            for (int c = lane; c < 2 * G; c += 32) m = max(m, __ldcg(p.sabs + c));
            m = __reduce_max_sync(0xffffffffu, m);
            int sh = 0;
            while ((m >> sh) >= 2048u) sh++;
            if (lane == 0) p.bin_sh[l] = sh;
        }
        // h of this layer was consumed in P2: clear it for layer l+2 (accumulated after By of l+1)
        if (cta == 0)
            for (int i = tid; i < r; i += NT) hcur[(int64_t)i * kHStride] = 0;
        // the other histogram buffer was last read in layer l-1's P3: clear it for layer l+1
        if (cta == G - 1)
            for (int i = tid; i < kHistW; i += NT) p.ghist[((l + 1) & 1) * kHistW + i] = 0;
        mbar_wait(&sel_bar, (uint32_t)(l & 1));
        STAMP(2);
        // Cut t (t = 0, 1, 2: the k16-th, (k16+k8)-th and k-th score in (score desc, id asc)
        // order, R3) is found by warp t: suffix scans of the 64 coarse then 64 fine histogram
        // bins locate the bin and the rank needed inside it.
        for (int t = warp; t < 3; t += NW) {
            if (tg(t) <= 0) continue;
            const int ca = hs[kBins + 63 - 2 * lane], cb = hs[kBins + 62 - 2 * lane];
            int inc = ca + cb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            int before = inc - ca - cb;  // count above this lane's first coarse bin
            int cbin = -1, need = 0;
            if (before < tg(t) && before + ca >= tg(t)) {
                cbin = 63 - 2 * lane;
                need = tg(t) - before;
            } else if (before + ca < tg(t) && before + ca + cb >= tg(t)) {
                cbin = 62 - 2 * lane;
                need = tg(t) - before - ca;
            }
            const unsigned who = __ballot_sync(0xffffffffu, cbin >= 0);
            if (!who) {  // histogram total < target: cannot happen with a consistent plan
                if (lane == 0) flag_error(p.err, 8u);
                continue;
            }
            const int src = __ffs(who) - 1;
            cbin = __shfl_sync(0xffffffffu, cbin, src);
            need = __shfl_sync(0xffffffffu, need, src);
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
        }
        __syncthreads();
        STAMP(3);
        auto id_of = [&](int e, int key) { return (e / RP) * rps + 255 - (key & 255); };  // e: run-array index
        // The steps below are warp-cooperative and compact (the layer loop's code does not fit
        // the instruction cache; straight-line single-thread code here is fetch-bound):
        // warp w takes runs c = w, w + NW, ...; lane j holds key e0 + j of the run.
        int *pcum = reinterpret_cast<int *>(S.ring + kCcOff);   // [G][4]: #keys >= K0, K1, K2
        int *pex = reinterpret_cast<int *>(S.ring + kExOff);    // [G][4]: list positions per tier
        {  // candidates: the (score, id) pairs of each cut bin -- the top of every sorted run
            int2 *cand = reinterpret_cast<int2 *>(S.ring + kCandOff);
            // value interval of each cut bin (bins 0 and 4095 are clamped: open-ended)
            int lo[3], hi[3], LO = 0x7fffffff;
#pragma unroll
            for (int t = 0; t < 3; t++) {
                const int b = cut_bin[t];
                lo[t] = b <= 0 ? -0x7fffffff : (b - 2048) * (1 << shl);
                hi[t] = b >= 4095 ? 0x7fffffff : (b - 2047) * (1 << shl) - 1;
                if (b < 0) {
                    lo[t] = 0x7fffffff;
                    hi[t] = (int)0x80000000;
                }
                LO = min(LO, lo[t]);
            }
            auto cand_add = [&](bool h0, bool h1, bool h2, int v, int n) {
                if (h0) {
                    const int at = atomicAdd(&ccnt[0], 1);
                    if (at < kCand) cand[at] = make_int2(v, n);
                }
                if (h1) {
                    const int at = atomicAdd(&ccnt[1], 1);
                    if (at < kCand) cand[kCand + at] = make_int2(v, n);
                }
                if (h2) {
                    const int at = atomicAdd(&ccnt[2], 1);
                    if (at < kCand) cand[2 * kCand + at] = make_int2(v, n);
                }
            };
            const int lo0 = lo[0], hi0 = hi[0], lo1 = lo[1], hi1 = hi[1], lo2 = lo[2], hi2 = hi[2];
            // thread (run c, cut t): two binary searches in the sorted run give the keys above
            // cut t's bin (all in cut t's prefix) and the bin's members (the candidates)
#pragma unroll 1
            for (int it = tid; it < 3 * G; it += NT) {
                const int t = it / G, c = it - t * G;
                if (cut_bin[t] < 0) {
                    if (t == 0) pcum[4 * c + 3] = 0;
                    pcum[4 * c + t] = 0;
                    continue;
                }
                const int nown = min(rps, F_r - c * rps);
                const int lt = t == 0 ? lo0 : (t == 1 ? lo1 : lo2), ht = t == 0 ? hi0 : (t == 1 ? hi1 : hi2);
                // #keys >= X in run c (keys descend); X as a 64-bit value (bin edges may be open)
                auto count_ge = [&](long long X) {
                    int a = 0, b = nown;
                    while (a < b) {
                        const int mid = (a + b) >> 1;
                        if ((long long)runkey(c, mid) >= X) a = mid + 1;
                        else b = mid;
                    }
                    return a;
                };
#if M2C_CAND_WALK
                const int ib = count_ge((long long)lt * 256);  // v >= lt
                int ia = ib;                                     // v > ht: the bin's members
                while (ia > 0 && (runkey(c, ia - 1) >> 8) <= ht) ia--;  // are few: walk up
#else
                const int ia = count_ge(((long long)ht + 1) * 256);  // v > ht
                const int ib = count_ge((long long)lt * 256);        // v >= lt
#endif
                pcum[4 * c + t] = ia;
                for (int e = ia; e < ib; e++) {  // the bin's members (few)
                    const int key = runkey(c, e);
                    cand_add(t == 0, t == 1, t == 2, key >> 8, c * rps + 255 - (key & 255));
                }
            }
            __syncthreads();
            STAMP(16);
            // exact rank of the candidates of cut t (warp t): the need-th in (score desc, id asc)
            for (int t = warp; t < 3; t += NW) {
                const int m = ncand[t];
                if (tg(t) <= 0 || m > kCand) continue;
                if (ccnt[t] != m && lane == 0) flag_error(p.err, 8u);
                const int2 c0 = lane < m ? cand[t * kCand + lane] : make_int2(0, 0);
                const int2 c1 = lane + 32 < m ? cand[t * kCand + lane + 32] : make_int2(0, 0);
                int r0 = 0, r1 = 0;
#pragma unroll 1
                for (int j = 0; j < m; j++) {
                    const int2 cj = cand[t * kCand + j];
                    r0 += (cj.x > c0.x) || (cj.x == c0.x && cj.y < c0.y);
                    r1 += (cj.x > c1.x) || (cj.x == c1.x && cj.y < c1.y);
                }
                const int want = cut_need[t] - 1;
                if (lane < m && r0 == want) {
                    cut_V[t] = c0.x;
                    cut_I[t] = c0.y;
                }
                if (lane + 32 < m && r1 == want) {
                    cut_V[t] = c1.x;
                    cut_I[t] = c1.y;
                }
                __syncwarp();
                // the bin's members ranked at or above the cut belong to its prefix
                if (lane < m && r0 <= want) atomicAdd(&pcum[4 * (c0.y / rps) + t], 1);
                if (lane + 32 < m && r1 <= want) atomicAdd(&pcum[4 * (c1.y / rps) + t], 1);
            }
            __syncthreads();
        }
        const bool degenerate = (tg(0) > 0 && ncand[0] > kCand) || (tg(1) > 0 && ncand[1] > kCand) ||
                                (tg(2) > 0 && ncand[2] > kCand);
        if (degenerate) {
            // degenerate (massive ties in one bin): binary searches with block-wide counts over
            // all keys (padding entries never count: their score is below -smax)
            for (int t = 0; t < 3; t++) {
                if (tg(t) <= 0 || ncand[t] <= kCand) continue;
                int lo = -p.smax, hi = p.smax;
                while (lo < hi) {  // largest V with #{s >= V} >= tg
                    const int mid = lo + (hi - lo + 1) / 2;
                    int c = 0;
                    for (int e = tid; e < G * RP; e += NT) c += (__ldcg(p.runs + e) >> 8) >= mid;
                    if (block_sum(c, red_i) >= tg(t)) lo = mid;
                    else hi = mid - 1;
                }
                const int V = lo;
                int c = 0;
                for (int e = tid; e < G * RP; e += NT) c += (__ldcg(p.runs + e) >> 8) > V;
                const int R = tg(t) - block_sum(c, red_i);
                int ilo = 0, ihi = F_r - 1;
                while (ilo < ihi) {  // smallest I with #{n <= I : s == V} >= R
                    const int mid = (ilo + ihi) >> 1;
                    int c2_ = 0;
                    for (int e = tid; e < G * RP; e += NT) {
                        const int key = __ldcg(p.runs + e);
                        c2_ += (key >> 8) == V && key != (int)0x80000000 && id_of(e, key) <= mid;
                    }
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
        // classify and compact.  The tier-t members of run c are a contiguous segment of it
        // (keys >= K_t(c), nested; K_t(c) is cut t's key as seen from c's local ids): ballots
        // count them per run, warp 0 scans the counts over runs into list positions, and the
        // few runs meeting this CTA's share of a tier list write its ids (ascending-id order
        // inside a segment = ascending local index).
        int n_items, c1, c2;
        {
            const int r0 = sm.rng[0], r1 = sm.rng[1], r2 = sm.rng[2], r3 = sm.rng[3], r4 = sm.rng[4],
                      r5 = sm.rng[5];
            const int off1 = r1 - r0, off2 = off1 + r3 - r2;
            c1 = off1;
            c2 = off2;
            n_items = off2 + r5 - r4;
            if (degenerate) {  // massive ties: exact per-run counts against the cut keys
            int *pK = pex;  // [G][4] per-run cut keys (pex is written only after they are used)
            for (int c = tid; c < G; c += NT) {  // cut t's key as seen from run c's local ids:
                int kq[3];                        // key >= K <=> s > V, or s == V and local <= loc
#pragma unroll
                for (int t = 0; t < 3; t++) {
                    const int V = cut_V[t], loc = cut_I[t] - c * rps;
                    kq[t] = cut_I[t] < 0 ? 0x7fffffff : (loc < 0 ? (V + 1) * 256 : V * 256 + 255 - min(loc, 255));
                }
                *reinterpret_cast<int4 *>(pK + 4 * c) = make_int4(kq[0], kq[1], kq[2], 0);
            }
            __syncthreads();
#pragma unroll 1
            for (int c = warp; c < G; c += NW) {
                const int nown = min(rps, F_r - c * rps);
                const int4 K = *reinterpret_cast<const int4 *>(pK + 4 * c);
                const int key = lane < nown ? ts[c * T + lane] : (int)0x80000000;
                int q2 = __popc(__ballot_sync(0xffffffffu, key >= K.z));
                int q1 = __popc(__ballot_sync(0xffffffffu, key >= K.y));
                int q0 = __popc(__ballot_sync(0xffffffffu, key >= K.x));
                if (q2 == 32 && nown > 32) {  // rare: the k-th cut is past key 32 of this run
#pragma unroll 1
                    for (int e0 = 32; e0 < nown; e0 += 32) {
                        const int e = e0 + lane;
                        const int k2 = e < nown ? runkey(c, e) : (int)0x80000000;
                        q2 += __popc(__ballot_sync(0xffffffffu, k2 >= K.z));
                        q1 += __popc(__ballot_sync(0xffffffffu, k2 >= K.y));
                        q0 += __popc(__ballot_sync(0xffffffffu, k2 >= K.x));
                        if (__shfl_sync(0xffffffffu, k2, 31) < K.z) break;
                    }
                }
                if (lane == 0) *reinterpret_cast<int4 *>(pcum + 4 * c) = make_int4(q0, q1, q2, 0);
            }
            }
            __syncthreads();
            STAMP(18);
            if (warp == 0) {  // exclusive scan of the per-run tier counts over runs
                constexpr int kSP = 5;  // runs per lane (G <= 160); loads issued together
                const int ca = lane * kSP;
                int4 qv[kSP];
#pragma unroll
                for (int u = 0; u < kSP; u++)
                    qv[u] = ca + u < G ? *reinterpret_cast<const int4 *>(pcum + 4 * (ca + u)) : make_int4(0, 0, 0, 0);
                int s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
                for (int u = 0; u < kSP; u++) {
                    s0 += qv[u].x;
                    s1 += qv[u].y - qv[u].x;
                    s2 += qv[u].z - qv[u].y;
                }
                int i0 = s0, i1 = s1, i2 = s2;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y0 = __shfl_up_sync(0xffffffffu, i0, o), y1 = __shfl_up_sync(0xffffffffu, i1, o),
                              y2 = __shfl_up_sync(0xffffffffu, i2, o);
                    if (lane >= o) {
                        i0 += y0;
                        i1 += y1;
                        i2 += y2;
                    }
                }
                int e0 = i0 - s0, e1 = i1 - s1, e2 = i2 - s2;
#pragma unroll
                for (int u = 0; u < kSP; u++) {
                    if (ca + u < G) *reinterpret_cast<int4 *>(pex + 4 * (ca + u)) = make_int4(e0, e1, e2, 0);
                    e0 += qv[u].x;
                    e1 += qv[u].y - qv[u].x;
                    e2 += qv[u].z - qv[u].y;
                }
                if (lane == 31 && (i0 != p.k16 || i1 != p.k8 || i2 != p.k4)) flag_error(p.err, 8u);
            }
            __syncthreads();
            STAMP(19);
            const int sg1 = p.k16, sg2 = p.k16 + p.k8;
            // work items: the (run, tier) segments that meet this CTA's share (thread per run)
            int *work = reinterpret_cast<int *>(S.ring + kWorkOff);  // [<= 3 G]
            if (tid == 0) ccnt[0] = 0;
            __syncthreads();
            for (int c = tid; c < G; c += NT) {
                const int4 q = *reinterpret_cast<const int4 *>(pcum + 4 * c);
                const int4 x = *reinterpret_cast<const int4 *>(pex + 4 * c);
                if (x.x < r1 && x.x + q.x > r0) work[atomicAdd(&ccnt[0], 1)] = 4 * c;
                if (x.y < r3 && x.y + q.y - q.x > r2) work[atomicAdd(&ccnt[0], 1)] = 4 * c + 1;
                if (x.z < r5 && x.z + q.z - q.y > r4) work[atomicAdd(&ccnt[0], 1)] = 4 * c + 2;
            }
            __syncthreads();
            const int nwork = ccnt[0];
#pragma unroll 1
            for (int w = warp; w < nwork; w += NW) {
                const int c = work[w] >> 2, t = work[w] & 3;
                const int4 q = *reinterpret_cast<const int4 *>(pcum + 4 * c);
                const int4 x = *reinterpret_cast<const int4 *>(pex + 4 * c);
                const int seg0 = t == 0 ? 0 : (t == 1 ? q.x : q.y), seg1 = t == 0 ? q.x : (t == 1 ? q.y : q.z);
                const int pa = t == 0 ? x.x : (t == 1 ? x.y : x.z);
                const int ra = t == 0 ? r0 : (t == 1 ? r2 : r4), rb = t == 0 ? r1 : (t == 1 ? r3 : r5);
                const int off = t == 0 ? 0 : (t == 1 ? off1 : off2);
                const int sg = t == 0 ? 0 : (t == 1 ? sg1 : sg2);
#pragma unroll 1
                for (int i0 = seg0; i0 < seg1; i0 += 32) {
                    const int i = i0 + lane;
                    const int lc = i < seg1 ? 255 - (runkey(c, i) & 255) : 0x40000000;
                    int rk = 0;  // members with a smaller id come first
#pragma unroll 1
                    for (int j = seg0; j < seg1; j++) rk += (255 - (runkey(c, j) & 255)) < lc;
                    const int pos = pa + rk;
                    if (i < seg1 && pos >= ra && pos < rb) {
                        S.loc[off + pos - ra] = c * rps + lc;
                        lst[sg + pos] = c * rps + lc;
                    }
                }
            }
            if (tid == 0)
                for (int t = 0; t < 3; t++) fa.pool[t] = Ld.pool[t];
            STAMP(11);
            fence_proxy_async();  // generic smem traffic in the ring precedes the TMA writes
            __syncthreads();
        }
        STAMP(5);
        if (p.select_only) break;  // the LRU/ATU chain: predictor + selection only; the lists
                                    // are out (the histogram is cleared by the next launch's prologue)

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
        // barrier By; meanwhile (warp 1, in TMA-queue order): this CTA's A^T chunks of layer
        // l+1 -> smem for R, then L2 prefetches: layer l+1's B slice and the previous token's
        // records of layer l+1, layer l+2's A^T chunks (staged at the next By)
        grid_sync(p.bar_flags, base + ++nbar, p.err, [&] {
            if (l + 1 < p.n_layers) {
                if ((threadIdx.x & 31) == 0 && cta < nchunk) {
                    fence_proxy_async();  // the FFN's generic reads of the ring precede the copy
                    const int nown = (nchunk - cta + G - 1) / G;
                    const uint32_t bytes = 32u * (uint32_t)r;
                    mbar_expect_tx(&at_bar, bytes * nown);
                    for (int q = 0; q < nown; q++)
                        bulk_g2s_plain(S.ring + kAtOff + q * bytes,
                                       p.layers[l + 1].At + (int64_t)(cta + q * G) * bytes, bytes, &at_bar);
                }
                prefetch_layers(p, l + 1, l + 2 < p.n_layers ? l + 2 : -1, l + 1);
            }
        });
        STAMP(7);
        if (l == p.n_layers - 1 && cta == G - 1)  // leave both histograms clear for the next token
            for (int i = tid; i < kHistW; i += NT) hist[i] = 0;

        // ================= R: fixed-order reduction + residual + next layer's h ==============
        {
            const bool more = l + 1 < p.n_layers;
            long long *hnext = p.hb + (int64_t)((l + 1) & 1) * r * kHStride;
            float(*rf)[33] = reinterpret_cast<float(*)[33]>(S.ring);
            const __half *xs_h = reinterpret_cast<const __half *>(S.xs);
            // the k_reduce order: virtual warp w sums rows w::32; two per pass, loads in flight
            auto reduce_chunk = [&](int e) {
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
            };
            const int P = p.nrank;
            const unsigned flag = round0 + (unsigned)l + 1u;
            const size_t row = (size_t)((flag - 1u) & 1u) * P;
            if (P > 1) {
                // the all-reduce fused into the reduction (§6.9): first every owned chunk of this
                // rank's y goes straight into every rank's exchange buffer as (flag | value)
                // 8-byte words (peer stores over NVLink; the flag is the exchange round, so a
                // word is complete when its flag matches -- no fences, no counters); the waits
                // follow in the loop below, so the round trips of a CTA's chunks overlap.
                for (int ch = cta; ch < nchunk; ch += G) {
                    const int e = ch * 32 + lane;
                    reduce_chunk(e);
                    __syncthreads();
                    if (warp == 0) {
                        float y = 0.f;
#pragma unroll
                        for (int w = 0; w < 32; w++) y += rf[w][lane];
                        const unsigned long long v = ((unsigned long long)flag << 32) | __float_as_uint(y);
                        for (int q = 0; q < P; q++) st_relaxed_sys_u64(p.xpeer[q] + (row + p.rank) * d + e, v);
                    }
                    __syncthreads();
                }
            }
            for (int ch = cta; ch < nchunk; ch += G) {
                const int e = ch * 32 + lane;
                if (P == 1) {
                    reduce_chunk(e);
                    __syncthreads();
                }
                if (warp == 0) {
                    float y = 0.f;
                    if (P == 1) {
#pragma unroll
                        for (int w = 0; w < 32; w++) y += rf[w][lane];
                    } else {
                        // every lane polls its element's P words in this rank's buffer and sums
                        // them in rank order.  Only the CTAs owning the same chunk on the P
                        // ranks meet: no cross-GPU barrier.
                        const unsigned long long *mine = p.xpeer[p.rank] + row * d + e;
                        for (int q = 0; q < P; q++) {
                            unsigned long long w = ld_relaxed_sys_u64(mine + (size_t)q * d);
                            if ((unsigned)(w >> 32) != flag &&
                                !(*reinterpret_cast<volatile unsigned *>(p.err) & 16u)) {
                                // (after one timeout no CTA waits again: a dead peer costs
                                // 5 s per token, not per chunk)
                                const unsigned long long t0 = gtimer();
                                do {
                                    w = ld_relaxed_sys_u64(mine + (size_t)q * d);
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
                    if (p.post_y) p.post_y[e] = y;  // split mode: this rank's y, to be all-reduced
                    else p.x[e] = xn;
                    if (more) {
                        bool bad = false;
                        int m, sh;
                        fp16_fixed(__half_as_ushort(xn), m, sh, bad);
                        if (bad) flag_error(p.err, 1u);
                        xm[lane] = m;
                        xsh[lane] = sh;
                    }
                }
                __syncthreads();
                if (more) {
                    if (ch == cta) mbar_wait(&at_bar, (uint32_t)(l & 1));  // A^T chunks staged at By
                    h_chunk(reinterpret_cast<const int8_t *>(S.ring + kAtOff) + (ch - cta) / G * 32 * r, r,
                            xm, xsh, hnext);
                    __syncthreads();
                }
            }
        }
        STAMP(8);
        if (l + 1 < p.n_layers) grid_sync(p.bar_flags, base + ++nbar, p.err);
    }
    STAMP(9);
#undef STAMP
    if (cta == 0 && tid == 0) {
        *p.bar_epoch = base + nbar;  // the next launch is stream-ordered
        if (p.nrank > 1) *p.rounds = round0 + (unsigned)p.n_layers;
    }
}

}  // namespace

size_t decode_layer_table_bytes(int n_layers) { return sizeof(DecLayer) * (size_t)n_layers; }
size_t decode_hist_bytes() { return sizeof(int) * 2 * (size_t)kHistW; }
// run prefix every CTA copies: ~2x a CTA's expected share of the active set, 16-B rows
// (the whole run: a probe past a partial prefix would stall its warp on an L2 load)
int decode_top_len(const m2c_ctx *c) {
    const int G = c->G, rps = (c->F_r + G - 1) / G;
    return rps | 1;
}
// all runs fit the ring behind the histogram scratch; run keys hold local indices < 255
int decode_max_F() { return 254 * 148 < (kRing - kSbufOff) / 4 - 4 * 148 ? 254 * 148 : (kRing - kSbufOff) / 4 - 4 * 148; }

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
        t[l].At = L.A;
        t[l].B = L.B;
        for (int k = 0; k < 3; k++) t[l].pool[k] = L.pool[k];
    }
    return cudaMemcpy(dev_table, t.data(), sizeof(DecLayer) * t.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_decode(m2c_ctx *c, __half *x, unsigned long long *prof, cudaStream_t st, int layer0,
                          int nl, const float *pre_y, float *post_y, int32_t *lists_out) {
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
    a.runs = c->dec_runs;
    a.T = decode_top_len(c);
    a.ghist = c->dec_hist;
    a.lists = lists_out ? lists_out : c->prev_ids + (size_t)layer0 * (c->plan.k > 0 ? c->plan.k : 1);
    a.select_only = lists_out != nullptr;
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
    // M2C_DECODE_PREFETCH (see prefetch_layers; a tuning / measurement knob, results are identical)
    {
        const char *ev = getenv("M2C_DECODE_PREFETCH");
        a.prefetch = ev ? atoi(ev) : 0;  // off: L2 prefetch traffic slows the latency-bound phases (tools/exp_prefetch.sh)
    }
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
    static const int pdl = [] {  // M2C_DECODE_PDL=0 disables (A/B knob; results identical)
        const char *ev = getenv("M2C_DECODE_PDL");
        return ev ? atoi(ev) : 1;
    }();
    if (lists_out && pdl) {  // select-only (LRU chain): overlap the launch with the previous kernel
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs = 2;
    }
    // <= 512 threads (d <= 4096): 128 registers per thread; else 64
    cudaError_t e = d / 8 <= 512 ? cudaLaunchKernelEx(&cfg, k_decode<512>, a)
                                 : cudaLaunchKernelEx(&cfg, k_decode<1024>, a);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

// k_ffn.cu -- a6: the list-driven FFN kernel (API path, LRU hits / misses); device code in
// ffn_dev.cuh (design notes there).
#include "ffn_dev.cuh"

namespace m2c {
namespace {


// ---- list-driven FFN (API path: m2c_sparse_ffn_forward, LRU hits / misses) --------------
// the miss FFN of the early-fill LRU engine consumes the staging area while k_fill (copy
// stream) is still filling it: entry e (tier segment offset included) is ready when
// ready[e] == tag (k_fill's release store after the record's bytes) or it was requantised
// (skip[e] >= 0: k_requant ran earlier on this stream)
struct RecWait {
    const int32_t *ready, *skip, *items, *step_ptr;
    int layer, seg[3], a0[3], c1, c2;
    uint32_t *err;
    __device__ __forceinline__ void operator()(int j) const {
        if (!ready) return;
        const int t = j < c1 ? 0 : (j < c2 ? 1 : 2);
        const int jj = j - (t == 0 ? 0 : (t == 1 ? c1 : c2));
        const int e = seg[t] + items[seg[t] + a0[t] + jj];
        if (skip && skip[e] >= 0) return;
        const int tag = fill_tag(*step_ptr, layer);
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ready + e) : "memory");
        if (v != tag) {
            const unsigned long long t0 = clock64();
            do {
                __nanosleep(100);
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ready + e) : "memory");
                if (clock64() - t0 > 4000000000ull) {  // ~2 s: a record that never lands
                    flag_error(err, 4u);
                    break;
                }
            } while (v != tag);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // (the TMA reads what it saw)
    }
};

__global__ void __launch_bounds__(1024, 1)
    k_ffn(FfnArgs a, int d, int act, const __half *__restrict__ x, const int32_t *__restrict__ items,
          const int32_t *__restrict__ counts, float *__restrict__ partial, RecWait w) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FfnShared sm;
    const SmemPtrs S = carve(smem);
    if (threadIdx.x == 0) ffn_init(sm, d);
    griddep_launch();
    griddep_wait();
    for (int c = threadIdx.x; c < d / 8; c += blockDim.x) S.xs[c] = reinterpret_cast<const uint4 *>(x)[c];
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
    FfnPipe pipe;
    if (w.ready) {
        w.items = items;
        w.c1 = c1;
        w.c2 = c2;
        for (int t = 0; t < 3; t++) w.seg[t] = a.seg[t];
        w.a0[0] = a0;
        w.a0[1] = a1;
        w.a0[2] = a2;
    }
    ffn_run(a, d, act, n_items, c1, c2, src, S.ring, S.xs, S.a, sm, pipe, partial, nullptr, w);
}

}  // namespace

cudaError_t init_ffn_attrs() {
    return cudaFuncSetAttribute(k_ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
}

cudaError_t launch_ffn(m2c_ctx *c, const LayerState &L, const __half *x, const int32_t *items,
                       const int32_t *counts, const m2c_tier_plan &p, float *partial,
                       cudaStream_t st, int wait_layer) {
    const int d = c->desc.d_model;
    FfnArgs a;
    fill_args(c, L, p, a);
    RecWait w = {};
    if (wait_layer >= 0) {  // (the early-fill engine's miss FFN)
        w.ready = c->mq_ready;
        w.skip = c->mq_src;
        w.step_ptr = c->ws.counts + 15;
        w.layer = wait_layer;
        w.err = c->ws.err;
    }
    cudaError_t e = launch_k(k_ffn, dim3(c->G), dim3(d / 8), kSmemBytes, st, a, d, c->desc.act, x,
                             items, counts, partial, w);
    c->launch_counter++;
    return e;
}

}  // namespace m2c

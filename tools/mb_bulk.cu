// mb_bulk.cu -- how fast can one CTA per SM pull scattered KB-sized records into smem?
//   A: 1-D TMA bulk copies (cp.async.bulk) of N records of S bytes, one mbarrier each
//   B: same with plain 16-B vector loads (ld.global.v4) by all threads into registers
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_bulk tools/mb_bulk.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const uint8_t *src, size_t stride_recs, int N, int S, unsigned long long *t_out, int evict_first) {
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ __align__(8) uint64_t bars[64];
    if (threadIdx.x == 0) {
        for (int i = 0; i < N; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) {
        uint64_t pol;
        if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        for (int i = 0; i < N; i++) {
            // record i of this CTA: spread over the buffer like gathered neurons
            const uint8_t *g = src + ((size_t)(blockIdx.x + i * gridDim.x) * stride_recs) * S;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[i])), "r"(S) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                         ::"r"(sa(ring + (size_t)i * S)), "l"(g), "r"(S), "r"(sa(&bars[i])), "l"(pol) : "memory");
        }
    }
    float acc = 0.f;
    for (int i = 0; i < N; i++) {
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(sa(&bars[i])) : "memory");
        acc += (float)ring[(size_t)i * S + threadIdx.x * 4];
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) { t_out[2 * blockIdx.x] = t0; t_out[2 * blockIdx.x + 1] = t1; }
    if (acc == 12345.f) t_out[0] = 0;
}

__global__ void k_ldg(const uint8_t *src, size_t stride_recs, int N, int S, unsigned long long *t_out) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int i = 0; i < N; i++) {
        const uint4 *g = reinterpret_cast<const uint4 *>(src + ((size_t)(blockIdx.x + i * gridDim.x) * stride_recs) * S);
        for (int c = threadIdx.x; c < S / 16; c += blockDim.x) {
            uint4 v = __ldg(g + c);
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) { t_out[2 * blockIdx.x] = t0; t_out[2 * blockIdx.x + 1] = t1; }
    if (acc.x == 0x12345) t_out[0] = acc.y;
}

int main() {
    size_t bytes = 4ull << 30;
    uint8_t *src;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMemset(src, 1, bytes));
    unsigned long long *t;
    CK(cudaMalloc(&t, 2 * 148 * 8));
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { int N, S; } cfgs[] = {{4, 24576}, {8, 12576}, {15, 6432}, {1, 24576}, {32, 6144}, {8, 24576}};
    for (auto c : cfgs) {
        for (int mode = 0; mode < 3; mode++) {
            size_t stride = 7;  // records apart (scattered gather)
            if ((size_t)(148 + c.N * 148) * stride * c.S > bytes) stride = 1;
            float best = 1e9;
            unsigned long long hs[296];
            for (int rep = 0; rep < 5; rep++) {
                CK(cudaMemset(src + bytes - 256 * 1024 * 1024ull, 0, 256 * 1024 * 1024ull));  // flush L2
                cudaEventRecord(e0);
                if (mode < 2) k_bulk<<<148, 512, c.N * c.S>>>(src, stride, c.N, c.S, t, mode);
                else k_ldg<<<148, 512>>>(src, stride, c.N, c.S, t);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) { best = ms; CK(cudaMemcpy(hs, t, sizeof(hs), cudaMemcpyDeviceToHost)); }
            }
            unsigned long long mn = ~0ull, mx = 0, sum = 0;
            for (int i = 0; i < 148; i++) {
                unsigned long long d = hs[2 * i + 1] - hs[2 * i];
                mn = d < mn ? d : mn; mx = d > mx ? d : mx; sum += d;
            }
            double totb = 148.0 * c.N * c.S;
            printf("%s N=%2d S=%6d: kernel %.2f us (%.0f GB/s)  per-CTA us min %.2f avg %.2f max %.2f\n",
                   mode == 0 ? "bulk(normal)" : mode == 1 ? "bulk(evict_first)" : "ldg.v4     ", c.N, c.S,
                   best * 1e3, totb / (best * 1e-3) / 1e9, mn / 1e3, sum / 148.0 / 1e3, mx / 1e3);
        }
    }
    return 0;
}

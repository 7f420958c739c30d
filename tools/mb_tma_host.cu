// mb_tma_host.cu -- can the TMA engine gather neuron records from pinned (UVA-mapped) host
// memory, and at what rate, next to the SM-driven warp-load gather of k_fill?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_tma_host tools/mb_tma_host.cu
//   /tmp/mb_tma_host [record_bytes] [records]
// A: warp per record, U x 16-B loads in flight per lane (k_fill's scheme), CTAs x 256 threads.
// B: per CTA, thread 0 streams its records host -> smem (cp.async.bulk, mbarrier) -> device
//    (cp.async.bulk.global.shared::cta, bulk_group), S stages of up to 32 KB in flight.
// C: cudaMemcpyAsync per record (DMA engine), for the PCIe peak of this access pattern.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int U>
__global__ void __launch_bounds__(256) k_warp(const uint8_t *host, uint8_t *dev, const int *idx, int n, int nb) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = gw; r < n; r += nw) {
        const uint4 *s = reinterpret_cast<const uint4 *>(host + (size_t)idx[r] * nb);
        uint4 *d = reinterpret_cast<uint4 *>(dev + (size_t)r * nb);
        const int n16 = nb / 16;
        for (int i = lane; i < n16; i += 32 * U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++) if (i + 32 * u < n16) v[u] = s[i + 32 * u];
#pragma unroll
            for (int u = 0; u < U; u++) if (i + 32 * u < n16) d[i + 32 * u] = v[u];
        }
    }
}

constexpr int kStage = 32768;
template <int S>
__global__ void __launch_bounds__(32) k_tma(const uint8_t *host, uint8_t *dev, const int *idx, int n, int nb) {
    extern __shared__ __align__(128) uint8_t buf[];  // S x kStage
    __shared__ __align__(8) uint64_t bar[S];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; s++)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the CTA's pieces: (record r, offset o) for r = blockIdx.x, +gridDim.x, ...; piece k -> stage k % S
    unsigned ph[S];
    for (int s = 0; s < S; s++) ph[s] = 0;
    int k = 0;
    for (int r = blockIdx.x; r < n; r += gridDim.x) {
        const uint8_t *src = host + (size_t)idx[r] * nb;
        for (int o = 0; o < nb; o += kStage, k++) {
            const int s = k % S, len = min(kStage, nb - o);
            if (k >= S) {  // the stage's previous store must have read the smem
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
            }
            uint8_t *b = buf + (size_t)s * kStage;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(len) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(b)), "l"(src + o), "r"(len), "r"(smem_u32(&bar[s])) : "memory");
            // wait for the OLDEST in-flight load (stage (k - S + 1) % S) and store it
            if (k >= S - 1) {
                const int ks = k - (S - 1), ss = ks % S;
                asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n}"
                             ::"r"(smem_u32(&bar[ss])), "r"(ph[ss]) : "memory");
                ph[ss] ^= 1u;
                // (recompute that piece's destination)
                // pieces are laid out in issue order: walk from the start of this CTA's list
                int rr = blockIdx.x, oo = 0;
                for (int kk = 0; kk < ks; kk++) { oo += kStage; if (oo >= nb) { oo = 0; rr += gridDim.x; } }
                const int l2 = min(kStage, nb - oo);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(dev + (size_t)rr * nb + oo), "r"(smem_u32(buf + (size_t)ss * kStage)), "r"(l2) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    // drain: the last S - 1 pieces
    for (int ks = max(0, k - (S - 1)); ks < k; ks++) {
        const int ss = ks % S;
        asm volatile("{\n\t.reg .pred P;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W2;\n}"
                     ::"r"(smem_u32(&bar[ss])), "r"(ph[ss]) : "memory");
        ph[ss] ^= 1u;
        int rr = blockIdx.x, oo = 0;
        for (int kk = 0; kk < ks; kk++) { oo += kStage; if (oo >= nb) { oo = 0; rr += gridDim.x; } }
        const int l2 = min(kStage, nb - oo);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dev + (size_t)rr * nb + oo), "r"(smem_u32(buf + (size_t)ss * kStage)), "r"(l2) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
    const int nb = argc > 1 ? atoi(argv[1]) : 30720;
    const int n = argc > 2 ? atoi(argv[2]) : 1024;
    const int pool = 13824;
    uint8_t *host;
    CK(cudaHostAlloc(&host, (size_t)pool * nb, cudaHostAllocMapped));
    for (size_t i = 0; i < (size_t)pool * nb; i++) host[i] = (uint8_t)(i * 2654435761u >> 13);
    uint8_t *hdev;
    CK(cudaHostGetDevicePointer((void **)&hdev, host, 0));
    uint8_t *dev, *ref;
    CK(cudaMalloc(&dev, (size_t)n * nb));
    CK(cudaMalloc(&ref, (size_t)n * nb));
    std::vector<int> idx(n);
    srand(7);
    for (int i = 0; i < n; i++) idx[i] = rand() % pool;
    int *didx;
    CK(cudaMalloc(&didx, 4 * n));
    CK(cudaMemcpy(didx, idx.data(), 4 * n, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double bytes = (double)n * nb;
    auto timeit = [&](const char *name, auto launch) {
        launch();
        CK(cudaStreamSynchronize(st));
        CK(cudaEventRecord(e0, st));
        for (int it = 0; it < 5; it++) launch();
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("%-28s %8.1f GB/s  (%d records x %d B, %.1f us per gather)\n", name, bytes * 5 / (ms * 1e-3) / 1e9,
               n, nb, ms * 1e3 / 5);
    };
    // C: DMA per record
    timeit("C cudaMemcpyAsync/record", [&] {
        for (int i = 0; i < n; i++)
            CK(cudaMemcpyAsync(ref + (size_t)i * nb, host + (size_t)idx[i] * nb, nb, cudaMemcpyHostToDevice, st));
    });
    for (int ctas : {32, 64}) {
        char nm[64];
        snprintf(nm, sizeof nm, "A warp loads U4 %d CTAs", ctas);
        timeit(nm, [&] { k_warp<4><<<ctas, 256, 0, st>>>(hdev, dev, didx, n, nb); });
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        std::vector<uint8_t> a((size_t)n * nb), b((size_t)n * nb);
        CK(cudaMemcpy(a.data(), dev, a.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), ref, b.size(), cudaMemcpyDeviceToHost));
        printf("   equal to DMA: %s\n", a == b ? "yes" : "NO");
    }
    CK(cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kStage));
    CK(cudaFuncSetAttribute(k_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * kStage));
    for (int ctas : {16, 32, 64}) {
        for (int S : {4, 6}) {
            char nm[64];
            snprintf(nm, sizeof nm, "B TMA S%d %d CTAs", S, ctas);
            CK(cudaMemset(dev, 0, (size_t)n * nb));
            timeit(nm, [&] {
                if (S == 4) k_tma<4><<<ctas, 32, 4 * kStage, st>>>(hdev, dev, didx, n, nb);
                else k_tma<6><<<ctas, 32, 6 * kStage, st>>>(hdev, dev, didx, n, nb);
            });
            cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) { printf("   TMA from host memory failed: %s\n", cudaGetErrorString(e)); return 0; }
            std::vector<uint8_t> a((size_t)n * nb), b((size_t)n * nb);
            CK(cudaMemcpy(a.data(), dev, a.size(), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(b.data(), ref, b.size(), cudaMemcpyDeviceToHost));
            printf("   equal to DMA: %s\n", a == b ? "yes" : "NO");
        }
    }
    return 0;
}

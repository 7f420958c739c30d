// Microbenchmark: grid-barrier latency on B200 (148 co-resident CTAs), three designs.
//   0: per-CTA flag words, one warp polls all flags (k_decode's design)
//   1: one counter, red.release.gpu.add arrive, ld.acquire poll of the counter
//   2: 16 sub-counters (CTA % 16), polled by 16 lanes
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_gridsync tools/mb_gridsync.cu
#include <cstdio>
#include <cuda_runtime.h>

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

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_nrank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// mode 3: cluster barrier, one arrival + one poller per cluster, cluster barrier to release
__global__ void k_bar_cluster(unsigned *buf, int iters, unsigned long long *out) {
    const unsigned ncl = gridDim.x / cluster_nrank();
    unsigned long long t0 = clock64();
    for (int it = 1; it <= iters; it++) {
        cluster_sync_all();
        if (cluster_rank() == 0 && threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(buf + 256) : "memory");
            while ((int)(ld_acquire(buf + 256) - (unsigned)(it * ncl)) < 0) {
            }
        }
        cluster_sync_all();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

template <int MODE>
__global__ void k_bar(unsigned *buf, int iters, unsigned long long *out) {
    const int G = gridDim.x;
    unsigned long long t0 = clock64();
    for (int it = 1; it <= iters; it++) {
        __syncthreads();
        if (threadIdx.x < 32) {
            if (MODE == 0) {
                if (threadIdx.x == 0)
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(buf + blockIdx.x), "r"((unsigned)it)
                                 : "memory");
                __syncwarp();
                for (;;) {
                    bool ok = true;
                    for (int i = threadIdx.x; i < G; i += 32) ok &= (int)(ld_relaxed(buf + i) - it) >= 0;
                    if (__all_sync(0xffffffffu, ok)) break;
                }
            } else if (MODE == 1) {
                if (threadIdx.x == 0)
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(buf + 256) : "memory");
                if (threadIdx.x == 0)
                    while ((int)(ld_acquire(buf + 256) - (unsigned)(it * G)) < 0) {
                    }
                __syncwarp();
            } else {
                const int sub = blockIdx.x & 15;
                const unsigned per = (G - sub + 15) / 16;  // CTAs mapped to this sub-counter
                if (threadIdx.x == 0)
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(buf + 512 + 32 * sub) : "memory");
                for (;;) {
                    bool ok = true;
                    if (threadIdx.x < 16) {
                        const unsigned n = (G - threadIdx.x + 15) / 16;
                        ok = (int)(ld_relaxed(buf + 512 + 32 * threadIdx.x) - (unsigned)(it * n)) >= 0;
                    }
                    if (__all_sync(0xffffffffu, ok)) break;
                }
                (void)per;
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned *buf;
    unsigned long long *out, h;
    cudaMalloc(&buf, 4 * 2048);
    cudaMalloc(&out, 8);
    const int iters = 2000;
    for (int mode = 0; mode < 3; mode++)
        for (int nt : {128, 512, 1024}) {
            cudaMemset(buf, 0, 4 * 2048);
            void *args[] = {&buf, (void *)&iters, &out};
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            void *fn = mode == 0 ? (void *)k_bar<0> : mode == 1 ? (void *)k_bar<1> : (void *)k_bar<2>;
            cudaEventRecord(e0);
            cudaError_t e = cudaLaunchCooperativeKernel(fn, sms, nt, args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("mode %d threads %4d: %s  %.3f us/barrier (event), %.0f cycles/barrier\n", mode, nt,
                   cudaGetErrorString(e), ms * 1e3 / iters, (double)h / iters);
        }
    for (int cs : {2, 4}) {
        for (int nt : {512, 1024}) {
            cudaMemset(buf, 0, 4 * 2048);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(sms);
            cfg.blockDim = dim3(nt);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int ncl = 0;
            cudaOccupancyMaxActiveClusters(&ncl, k_bar_cluster, &cfg);
            if (ncl * cs < sms) {
                printf("cluster %d threads %4d: only %d clusters co-resident, skipped\n", cs, nt, ncl);
                continue;
            }
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t e = cudaLaunchKernelEx(&cfg, k_bar_cluster, buf, iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("cluster %d threads %4d (%d clusters fit): %s  %.3f us/barrier\n", cs, nt, ncl,
                   cudaGetErrorString(e), ms * 1e3 / iters);
        }
    }
    return 0;
}

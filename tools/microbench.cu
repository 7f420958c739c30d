// microbench.cu -- B200 latency microbenchmarks that shape the decode-kernel design:
//   1. dependent empty-kernel chain in a CUDA graph, with and without PDL (per-hop cost)
//   2. persistent kernel with software grid barriers (per-barrier cost), 148 x {256,512} thr
//   3. int64 fixed-point atomics (red.global.add.u64) throughput, 148 CTAs x 4096 adds
//   4. zero-copy reads of pinned host memory from a kernel (H2D via SMs)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_empty(int *p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0]++;
}

__device__ __forceinline__ void grid_barrier(unsigned *count, volatile unsigned *gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = *gen;
        __threadfence();
        unsigned arrived = atomicAdd(count, 1u);
        if (arrived == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned *)gen, 1u);
        } else {
            while (*gen == g) { }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_barriers(unsigned *count, unsigned *gen, int n, long long *cycles) {
    long long t0 = clock64();
    for (int i = 0; i < n; i++) grid_barrier(count, gen, gridDim.x);
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = clock64() - t0;
}

__global__ void k_fixed_atomics(unsigned long long *acc, int d, int reps) {
    for (int r = 0; r < reps; r++)
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
            long long v = (long long)(blockIdx.x * 7 + i);
            asm volatile("red.global.add.u64 [%0], %1;" :: "l"(acc + i), "l"(v) : "memory");
        }
}

__global__ void k_vec_atomics(float *acc, int d, int reps) {
    for (int r = 0; r < reps; r++)
        for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(acc + i),
                         "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f) : "memory");
        }
}

__global__ void k_zero_copy(const uint4 *src, uint4 *dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int *dp;
    CK(cudaMalloc(&dp, 64));
    // 1. chain of N dependent empty kernels in a graph
    for (int pdl = 0; pdl < 2; pdl++)
        for (int grid : {1, 148}) {
            const int N = 200;
            cudaGraph_t g;
            cudaGraphExec_t ge;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            for (int i = 0; i < N; i++) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                a[0].val.programmaticStreamSerializationAllowed = pdl;
                cfg.attrs = a;
                cfg.numAttrs = 1;
                CK(cudaLaunchKernelEx(&cfg, k_empty, dp));
            }
            CK(cudaStreamEndCapture(s, &g));
            CK(cudaGraphInstantiate(&ge, g, 0));
            for (int w = 0; w < 3; w++) CK(cudaGraphLaunch(ge, s));
            cudaEventRecord(e0, s);
            for (int w = 0; w < 10; w++) CK(cudaGraphLaunch(ge, s));
            cudaEventRecord(e1, s);
            CK(cudaStreamSynchronize(s));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("chain: pdl=%d grid=%3d  %.3f us per dependent kernel\n", pdl, grid, ms * 1e3 / (10 * N));
        }
    // 2. grid barriers
    unsigned *cnt;
    long long *cyc;
    CK(cudaMalloc(&cnt, 256));
    CK(cudaMalloc(&cyc, 8));
    for (int threads : {256, 512}) {
        CK(cudaMemset(cnt, 0, 256));
        const int n = 1000;
        cudaEventRecord(e0, s);
        void *args[] = {&cnt, nullptr, (void *)&n, &cyc};
        unsigned *gen = cnt + 32;
        args[1] = &gen;
        CK(cudaLaunchCooperativeKernel((void *)k_barriers, dim3(148), dim3(threads), args, 0, s));
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("grid barrier: 148 x %d thr: %.3f us per barrier (%.0f cycles)\n", threads, ms * 1e3 / n, (double)c / n);
    }
    // 3. atomics
    unsigned long long *acc;
    CK(cudaMalloc(&acc, 8 * 8192));
    for (int d : {4096, 8192}) {
        k_fixed_atomics<<<148, 512, 0, s>>>(acc, d, 1);
        cudaEventRecord(e0, s);
        k_fixed_atomics<<<148, 512, 0, s>>>(acc, d, 10);
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("red.u64: 148 CTAs x %d: %.3f us per round\n", d, ms * 1e3 / 10);
        k_vec_atomics<<<148, 512, 0, s>>>((float *)acc, d, 1);
        cudaEventRecord(e0, s);
        k_vec_atomics<<<148, 512, 0, s>>>((float *)acc, d, 10);
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("red.v4.f32: 148 CTAs x %d: %.3f us per round\n", d, ms * 1e3 / 10);
    }
    // 4. zero-copy host reads
    size_t bytes = 256ull << 20;
    void *h, *dd;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&dd, bytes));
    for (int grid : {16, 32, 64, 148, 296}) {
        k_zero_copy<<<grid, 512, 0, s>>>((const uint4 *)h, (uint4 *)dd, bytes / 16);
        cudaEventRecord(e0, s);
        k_zero_copy<<<grid, 512, 0, s>>>((const uint4 *)h, (uint4 *)dd, bytes / 16);
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("zero-copy H2D kernel read: grid %d: %.1f GB/s\n", grid, bytes / (ms * 1e-3) / 1e9);
    }
    cudaEventRecord(e0, s);
    CK(cudaMemcpyAsync(dd, h, bytes, cudaMemcpyHostToDevice, s));
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cudaMemcpyAsync H2D 256MB: %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);
    return 0;
}

// Microbenchmark: grid-barrier variants on B200 (148 co-resident CTAs, one per SM), measured
// in a loop of back-to-back barriers, optionally with every thread storing to global memory
// before each barrier (the release then has pending writes to order, as in k_decode).
//   1: red.release.gpu.add arrive, ld.acquire poll                 (k_decode today)
//   2: red.release arrive, ld.relaxed poll, one fence.acq_rel after
//   3: fence.acq_rel + red.relaxed arrive, ld.relaxed poll, fence.acq_rel after
//   4: red.relaxed + ld.relaxed, no fences (latency floor; NOT memory-safe)
//   5: atom.add.acq_rel arrive (returns old), last arriver st.release a flag word on another
//      line, the rest poll the flag with ld.relaxed + fence after
//   6: like 2, poller is lane 0 of every warp (no trailing __syncthreads)
//   7: no atomics: every CTA st.release its own flag line; warp 0 polls all G flags (ld.relaxed,
//      lanes over CTAs), one fence.acq_rel after
//   8: arrival counters split 8 ways (cta % 8, own lines); thread 0 polls the 8 sums
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_gridsync2 tools/mb_gridsync2.cu
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

template <int MODE>
__global__ void k_bar(unsigned *buf, float *sink, int iters, int nstore, unsigned long long *out) {
    const int G = gridDim.x;
    unsigned *cnt = buf + 256, *flag = buf + 1024;
    unsigned long long t0 = clock64();
    for (int it = 1; it <= iters; it++) {
        for (int s = 0; s < nstore; s++)
            sink[((size_t)blockIdx.x * nstore + s) * blockDim.x + threadIdx.x] = (float)it;
        if (MODE == 6) {
            __syncthreads();
            if ((threadIdx.x & 31) == 0) {
                if (threadIdx.x == 0)
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while ((int)(ld_relaxed(cnt) - (unsigned)(it * G)) < 0) {
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            __syncwarp();
            continue;
        }
        if (MODE == 7) {
            __syncthreads();
            unsigned *fl = buf + 2048;  // flags, one per CTA, 64 B apart? (index * 16 u32)
            if (threadIdx.x == 0)
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(fl + 16 * blockIdx.x), "r"((unsigned)it) : "memory");
            if (threadIdx.x < 32) {
                for (int c = threadIdx.x; c < G; c += 32)
                    while ((int)(ld_relaxed(fl + 16 * c) - (unsigned)it) < 0) {
                    }
                __syncwarp();
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            __syncthreads();
            continue;
        }
        if (MODE == 8) {
            __syncthreads();
            if (threadIdx.x == 0)
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + 32 * (blockIdx.x & 7)) : "memory");
            if (threadIdx.x < 8) {
                const unsigned want8 = (unsigned)(it * ((G - threadIdx.x + 7) / 8));
                while ((int)(ld_relaxed(cnt + 32 * threadIdx.x) - want8) < 0) {
                }
                __syncwarp(0xffu);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            __syncthreads();
            continue;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned want = (unsigned)(it * G);
            if (MODE == 1) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while ((int)(ld_acquire(cnt) - want) < 0) {
                }
            } else if (MODE == 2) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while ((int)(ld_relaxed(cnt) - want) < 0) {
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (MODE == 3) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while ((int)(ld_relaxed(cnt) - want) < 0) {
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (MODE == 4) {
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while ((int)(ld_relaxed(cnt) - want) < 0) {
                }
            } else if (MODE == 5) {
                unsigned old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
                if (old == want - 1) {
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"((unsigned)it) : "memory");
                } else {
                    while ((int)(ld_relaxed(flag) - (unsigned)it) < 0) {
                    }
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *buf;
    float *sink;
    unsigned long long *out, h;
    cudaMalloc(&buf, 4 * 8192);
    cudaMalloc(&sink, (size_t)sms * 8 * 1024 * 4);
    cudaMalloc(&out, 8);
    const int iters = 2000;
    void *fns[9] = {nullptr, (void *)k_bar<1>, (void *)k_bar<2>, (void *)k_bar<3>,
                    (void *)k_bar<4>, (void *)k_bar<5>, (void *)k_bar<6>, (void *)k_bar<7>, (void *)k_bar<8>};
    for (int nstore : {0, 8})
        for (int mode = 1; mode <= 8; mode++)
            for (int nt : {512, 1024}) {
                cudaMemset(buf, 0, 4 * 8192);
                void *args[] = {&buf, &sink, (void *)&iters, (void *)&nstore, &out};
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaError_t e = cudaLaunchCooperativeKernel(fns[mode], sms, nt, args, 0, 0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
                printf("mode %d threads %4d stores/thread %d: %s  %.3f us/barrier (event), %.0f cycles\n", mode,
                       nt, nstore, cudaGetErrorString(e), ms * 1e3 / iters, (double)h / iters);
            }
    return 0;
}

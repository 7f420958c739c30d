// mc_probe.cu -- can this box build an NVLS multicast object and run multimem.* on it?
// One device: a multicast group of 1, 2 MB bound, multimem.red.add.f32 / multimem.ld_reduce.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
__global__ void k_mm(float *mc, float *uc, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(mc + i), "f"(1.5f) : "memory");
    }
    __syncthreads();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (i < n) {
        float v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + i) : "memory");
        uc[n + i] = v;
    }
}
int main() {
    CK(cuInit(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    int mc = 0; CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("multicast supported: %d\n", mc);
    CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
    if (!mc) return 0;
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1; prop.size = 2 << 20;
    size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    prop.size = ((prop.size + gran - 1) / gran) * gran;
    printf("granularity %zu, size %zu\n", gran, prop.size);
    CUmemGenericAllocationHandle mch;
    const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
    CUresult rr = CUDA_ERROR_UNKNOWN;
    int hi = 0;
    for (; hi < 3; hi++) {
        prop.handleTypes = hts[hi];
        rr = cuMulticastCreate(&mch, &prop);
        const char *es; cuGetErrorString(rr, &es);
        printf("cuMulticastCreate(handleTypes=%d) -> %s\n", (int)hts[hi], es);
        if (rr == CUDA_SUCCESS) break;
    }
    if (rr != CUDA_SUCCESS) return 1;
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
    CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, prop.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mem, 0, prop.size, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0)); CK(cuMemMap(uc, prop.size, 0, mem, 0));
    CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0)); CK(cuMemMap(mcp, prop.size, 0, mch, 0));
    CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, prop.size, &ad, 1)); CK(cuMemSetAccess(mcp, prop.size, &ad, 1));
    const int n = 4096;
    cudaMemset((void *)uc, 0, 8 * n);
    k_mm<<<n / 256, 256>>>((float *)mcp, (float *)uc, n);
    cudaError_t e = cudaDeviceSynchronize();
    float h[2];
    cudaMemcpy(h, (void *)uc, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h + 1, (char *)uc + 4 * n, 4, cudaMemcpyDeviceToHost);
    printf("kernel: %s; unicast[0] after multimem.red = %g, ld_reduce = %g (expect 1.5, 1.5)\n", cudaGetErrorString(e), h[0], h[1]);
    return 0;
}

// mc_test.cu — does NVLS multicast work on this box with one device?  (measurement tool)
// Creates a 1-device multicast object, binds a physical allocation, maps the multicast
// VA and a unicast VA, runs multimem.red.add.v4.f32 from a kernel and reads the result.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mc tools/mc_test.cu -lcuda && /tmp/mc
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
    printf("%s failed: %s\n", #x, s); return 1; } } while (0)

__global__ void red(float* mc, int n) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i + 4 <= n) {
        const float a = 1.0f + i, b = 2.0f, c = 3.0f, d = 4.0f;
        asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                     :: "l"(mc + i), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
    }
}

int main() {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    int mcs = 0;
    CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("multicast supported: %d\n", mcs);
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    mp.size = 2 << 20;
    CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t size = ((size_t)(4 << 20) + gran - 1) / gran * gran;
    mp.size = size;
    printf("granularity %zu size %zu\n", gran, size);
    CUmemGenericAllocationHandle mc;
    CUresult cr = cuMulticastCreate(&mc, &mp);
    if (cr != CUDA_SUCCESS) {
        const unsigned long long types[3] = {0, CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
        for (int t = 0; t < 3 && cr != CUDA_SUCCESS; ++t) {
            for (int nd = 1; nd <= 2 && cr != CUDA_SUCCESS; ++nd) {
                mp.handleTypes = types[t];
                mp.numDevices = nd;
                cr = cuMulticastCreate(&mc, &mp);
                const char* es;
                cuGetErrorString(cr, &es);
                printf("cuMulticastCreate handleTypes=%llu numDevices=%d -> %s\n", types[t], nd, es);
            }
        }
        if (cr != CUDA_SUCCESS) return 1;
    }
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
    CUdeviceptr uva, mva;
    CK(cuMemAddressReserve(&uva, size, gran, 0, 0));
    CK(cuMemMap(uva, size, 0, mem, 0));
    CK(cuMemAddressReserve(&mva, size, gran, 0, 0));
    CK(cuMemMap(mva, size, 0, mc, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uva, size, &acc, 1));
    CK(cuMemSetAccess(mva, size, &acc, 1));
    const int n = 1 << 16;
    cudaMemset((void*)uva, 0, n * 4);
    red<<<n / 4 / 256, 256>>>((float*)mva, n);
    red<<<n / 4 / 256, 256>>>((float*)mva, n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    float h[8];
    cudaMemcpy(h, (void*)uva, sizeof(h), cudaMemcpyDeviceToHost);
    printf("result: %g %g %g %g %g %g %g %g (expect 2 4 6 8 10 4 6 8)\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    return 0;
}

// multicast_probe.cu — does this box support NVLink SHARP multicast objects
// (cuMulticastCreate) for the visible GPU(s)?  Measurement tool only.
#include <cuda.h>
#include <cstdio>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); \
    printf("%s -> %d (%s)\n", #x, (int)r, s); return 1; } } while (0)

__global__ void mc_store(float *mc, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(mc + i), "f"((float)i) : "memory");
}

int main() {
    CK(cuInit(0));
    int ndev = 0;
    CK(cuDeviceGetCount(&ndev));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("devices %d, multicast supported %d\n", ndev, mc);
    if (!mc) return 0;
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    prop.size = 1 << 21;
    CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    prop.size = ((size_t)(1 << 21) + gran - 1) / gran * gran;
    printf("granularity %zu size %zu\n", gran, prop.size);
    CUmemGenericAllocationHandle mch;
    CK(cuMulticastCreate(&mch, &prop));
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, prop.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mem, 0, prop.size, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0));
    CK(cuMemMap(uc, prop.size, 0, mem, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, prop.size, &acc, 1));
    CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0));
    CK(cuMemMap(mcp, prop.size, 0, mch, 0));
    CK(cuMemSetAccess(mcp, prop.size, &acc, 1));
    const int n = 1 << 18;
    mc_store<<<n / 256, 256>>>((float *)mcp, n);
    CK(cuCtxSynchronize());
    float h[4];
    CK(cuMemcpyDtoH(h, uc + 4 * 1000, 16));
    printf("unicast view after multimem.st: %g %g %g %g (expect 1000..1003)\n", h[0], h[1], h[2], h[3]);
    return 0;
}

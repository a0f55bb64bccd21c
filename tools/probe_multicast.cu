// Probe: is NVLS multicast (multimem.st) usable on this box?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_multicast tools/probe_multicast.cu -lcuda
//
// Queries CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, tries cuMulticastCreate
// for 1 and 2 devices with every handle type, and — when an object can be
// created — binds one device allocation, maps the multicast address and
// checks that a multimem.st.v4.f32 store lands in the unicast view.
// On the one-GPU gpurun box of this build (r3): multicast_supported 1, fabric
// handles 1, but cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE for every
// combination, so the multicast epilogue of DESIGN.md section 6 cannot be
// validated here.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#define CK(x)                                            \
    do {                                                 \
        CUresult r_ = (x);                               \
        if (r_ != CUDA_SUCCESS) {                        \
            const char* s_ = nullptr;                    \
            cuGetErrorString(r_, &s_);                   \
            printf("%s -> %s\n", #x, s_ ? s_ : "?");     \
            return 1;                                    \
        }                                                \
    } while (0)

__global__ void mc_store(float* mc, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i * 4 < n) {
        const float a = i * 4.f, b = a + 1, c = a + 2, d = a + 3;
        asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i * 4), "f"(a), "f"(b),
                     "f"(c), "f"(d)
                     : "memory");
    }
}

int main() {
    CK(cuInit(0));
    int ndev = 0;
    CK(cuDeviceGetCount(&ndev));
    printf("devices %d\n", ndev);
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc = 0, fab = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("multicast_supported %d fabric_handle %d\n", mc, fab);
    if (!mc) return 0;
    cudaSetDevice(0);
    cudaFree(0);

    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof mp);
    mp.numDevices = 1;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    printf("mc granularity %zu\n", gran);
    const size_t size = gran;
    mp.size = size;
    const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE,
                                              CU_MEM_HANDLE_TYPE_FABRIC};
    for (int nd = 1; nd <= 2; ++nd)
        for (int h = 0; h < 3; ++h) {
            CUmulticastObjectProp q = mp;
            q.numDevices = nd;
            q.handleTypes = hts[h];
            CUmemGenericAllocationHandle t;
            const CUresult r = cuMulticastCreate(&t, &q);
            const char* es = nullptr;
            cuGetErrorString(r, &es);
            printf("create numDevices=%d handleType=%d -> %s\n", nd, static_cast<int>(hts[h]), es ? es : "?");
            if (r == CUDA_SUCCESS) cuMemRelease(t);
        }

    CUmemGenericAllocationHandle mch;
    CK(cuMulticastCreate(&mch, &mp));
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap;
    memset(&ap, 0, sizeof ap);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle mh;
    CK(cuMemCreate(&mh, size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mh, 0, size, 0));
    CUdeviceptr uc = 0, mcva = 0;
    CK(cuMemAddressReserve(&uc, size, gran, 0, 0));
    CK(cuMemMap(uc, size, 0, mh, 0));
    CK(cuMemAddressReserve(&mcva, size, gran, 0, 0));
    CK(cuMemMap(mcva, size, 0, mch, 0));
    CUmemAccessDesc ad;
    ad.location = ap.location;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, size, &ad, 1));
    CK(cuMemSetAccess(mcva, size, &ad, 1));
    cudaMemset(reinterpret_cast<void*>(uc), 0, 4096);
    mc_store<<<1, 256>>>(reinterpret_cast<float*>(mcva), 1024);
    const cudaError_t e = cudaDeviceSynchronize();
    float h[8];
    cudaMemcpy(h, reinterpret_cast<void*>(uc), sizeof h, cudaMemcpyDeviceToHost);
    printf("sync %s; unicast view after multimem.st: %g %g %g %g %g\n", cudaGetErrorString(e), h[0], h[1], h[2], h[3],
           h[5]);
    return 0;
}

// Probe: NVLS multicast on this box (one visible GPU).  Creates a multicast object for one
// device, binds physical memory, maps the multicast address and stores through it with
// multimem.st; the unicast mapping must then hold the values.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define CKD(x)                                                                  \
    do {                                                                        \
        CUresult r_ = (x);                                                      \
        if (r_ != CUDA_SUCCESS) {                                               \
            const char *s_ = nullptr;                                           \
            cuGetErrorString(r_, &s_);                                          \
            printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?");           \
            return 1;                                                           \
        }                                                                       \
    } while (0)

__global__ void mc_store(uint32_t *mc, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n / 4) {
        uint32_t a = 4 * i, b = 4 * i + 1, c = 4 * i + 2, d = 4 * i + 3;
        asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "r"(a), "r"(b), "r"(c),
                     "r"(d)
                     : "memory");
    }
}

int main() {
    CKD(cuInit(0));
    CUdevice dev;
    CKD(cuDeviceGet(&dev, 0));
    int mc = -1, fd = -1, fab = -1, vmm = -1;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
    printf("multicast=%d posix_fd=%d fabric=%d vmm=%d\n", mc, fd, fab, vmm);
    cudaSetDevice(0);
    cudaFree(0);
    if (!mc) return 0;
    const size_t want = 4 << 20;
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.size = want;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CKD(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    size_t sz = (want + gran - 1) / gran * gran;
    mp.size = sz;
    printf("mc granularity %zu size %zu\n", gran, sz);
    CUmemGenericAllocationHandle mch;
    {
        const int hts[3] = {0, (int)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (int)CU_MEM_HANDLE_TYPE_FABRIC};
        for (int nd = 1; nd <= 2; nd++)
            for (int h = 0; h < 3; h++)
                for (int small = 0; small < 2; small++) {
                    CUmulticastObjectProp q = mp;
                    q.numDevices = nd;
                    q.handleTypes = (unsigned long long)hts[h];
                    size_t g2 = 0;
                    cuMulticastGetGranularity(&g2, &q, CU_MULTICAST_GRANULARITY_MINIMUM);
                    q.size = small ? g2 : sz;
                    CUmemGenericAllocationHandle t;
                    CUresult r = cuMulticastCreate(&t, &q);
                    printf("create nd=%d ht=%d size=%zu (min gran %zu) -> %d\n", nd, hts[h], q.size, g2, (int)r);
                    if (r == CUDA_SUCCESS) cuMemRelease(t);
                }
    }
    mp.handleTypes = 0;
    CKD(cuMulticastCreate(&mch, &mp));
    CKD(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
    size_t ugran = 0;
    CKD(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    printf("unicast granularity %zu\n", ugran);
    CUmemGenericAllocationHandle ph;
    CKD(cuMemCreate(&ph, sz, &ap, 0));
    CKD(cuMulticastBindMem(mch, 0, ph, 0, sz, 0));
    CUdeviceptr uva, mva;
    CKD(cuMemAddressReserve(&uva, sz, gran, 0, 0));
    CKD(cuMemMap(uva, sz, 0, ph, 0));
    CKD(cuMemAddressReserve(&mva, sz, gran, 0, 0));
    CKD(cuMemMap(mva, sz, 0, mch, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = 0;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CKD(cuMemSetAccess(uva, sz, &ad, 1));
    CKD(cuMemSetAccess(mva, sz, &ad, 1));
    const int n = (int)(sz / 4);
    cudaMemset((void *)uva, 0, sz);
    mc_store<<<(n / 4 + 255) / 256, 256>>>((uint32_t *)mva, n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    uint32_t *h = (uint32_t *)malloc(sz);
    cudaMemcpy(h, (void *)uva, sz, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; i++) bad += h[i] != (uint32_t)i;
    printf("mismatches %d of %d\n", bad, n);
    // timing: multicast stores vs plain stores of the same size
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int it = 0; it < 20; it++) mc_store<<<(n / 4 + 255) / 256, 256>>>((uint32_t *)mva, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("multimem.st %zu bytes: %.2f us/launch, %.1f GB/s\n", sz, ms * 1e3 / 20, sz / (ms * 1e-3 / 20) / 1e9);
    int fdh = -1;
    CUresult r = cuMemExportToShareableHandle(&fdh, mch, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    printf("export mc handle to fd: %d (fd %d)\n", (int)r, fdh);
    printf("OK\n");
    return 0;
}

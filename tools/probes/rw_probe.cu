// Probe: HBM read-only, write-only and 1:1 copy bandwidth vs size on one B200 -- the
// denominators behind the write-heavy (1 read : 8 writes) single-GPU allgather.  Grid-stride
// 16-B accesses at full occupancy; write-only also as TMA bulk stores of a zeroed stage.
// Prints us per launch (20 back-to-back launches, events) and GB/s of the bytes touched.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void k_read(const uint4 *__restrict__ a, uint64_t n, uint32_t *sink) {
    uint32_t x = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(a + i);
        x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x12345678u) *sink = x;
}
__global__ void k_write(uint4 *__restrict__ a, uint64_t n) {
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        __stcs(a + i, v);
}
__global__ void k_copy(const uint4 *__restrict__ a, uint4 *__restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}
// 1 read : F writes (the allgather's fan-out), grid-stride over the source
template <int F>
__global__ void k_fan(const uint4 *__restrict__ a, uint4 *__restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(a + i);
#pragma unroll
        for (int f = 0; f < F; f++) b[(uint64_t)f * n + i] = v;
    }
}
// write-only through TMA bulk stores: each CTA stores a 16 KiB zeroed stage over its chunks
__global__ void k_write_tma(char *a, uint64_t nch) {
    extern __shared__ __align__(128) char st[];
    for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(st)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(st);
        int k = 0;
        for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x, k++) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a + c * 16384), "r"(s), "r"(16384) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (k >= 8) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const uint64_t maxN = 2048ull << 20;
    char *a, *b;
    uint32_t *sink;
    CK(cudaMalloc(&a, maxN));
    CK(cudaMalloc(&b, maxN));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(a, 1, maxN));
    CK(cudaMemset(b, 1, maxN));
    CK(cudaFuncSetAttribute(k_write_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int grid = 148 * 4, tpb = 512;
    printf("# MiB = bytes touched per launch; GB/s of bytes touched\n");
    for (uint64_t mib : {32ull, 64ull, 128ull, 256ull, 512ull, 1024ull, 2048ull}) {
        const uint64_t N = mib << 20;
        double r[6];
        for (int mode = 0; mode < 6; mode++) {
            auto go = [&]() {
                if (mode == 0) k_read<<<grid, tpb>>>((const uint4 *)a, N / 16, sink);
                if (mode == 1) k_write<<<grid, tpb>>>((uint4 *)a, N / 16);
                if (mode == 2) k_write_tma<<<148 * 2, 32, 16384>>>(a, N / 16384);
                if (mode == 3) k_copy<<<grid, tpb>>>((const uint4 *)a, (uint4 *)b, N / 32);
                if (mode == 4) k_fan<8><<<grid, tpb>>>((const uint4 *)a, (uint4 *)b, N / 16 / 9);
                if (mode == 5) k_fan<2><<<grid, tpb>>>((const uint4 *)a, (uint4 *)b, N / 16 / 3);
            };
            for (int i = 0; i < 3; i++) go();
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            for (int i = 0; i < 20; i++) go();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            r[mode] = (double)N / (ms * 1e-3 / 20) / 1e9;
        }
        printf("%5llu MiB: read %.0f  write %.0f  write_tma %.0f  copy %.0f  fan1:8 %.0f  fan1:2 %.0f GB/s\n",
               (unsigned long long)mib, r[0], r[1], r[2], r[3], r[4], r[5]);
    }
    return 0;
}

// HBM probe (measurement tool, not product): what a B200 sustains for the access mixes the
// mpxa kernels produce -- write-only, read-only, 1:1 copy (LSU and TMA bulk), and a 1:8
// fan-out copy (allgather direct).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_write(uint4 *d, size_t n) {
    uint4 v = make_uint4(1, 2, 3, 4);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = v;
}
__global__ void k_read(const uint4 *s, size_t n, uint32_t *sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(s + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}
__global__ void k_copy(uint4 *d, const uint4 *s, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = __ldcs(s + i);
}
__global__ void k_fan8(uint4 *d, const uint4 *s, size_t n) {   // d = 8 copies of s
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(s + i);
#pragma unroll
        for (int k = 0; k < 8; k++) d[k * n + i] = v;
    }
}
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// TMA bulk copy: one thread per CTA streams chunks through smem (nstage x chunk)
template <int S, int C>
__global__ void k_tma(char *d, const char *s, size_t bytes, int fan) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[S];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < S; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    size_t per = (bytes / gridDim.x) / C * C;
    const char *src = s + per * blockIdx.x;
    char *dst = d + per * blockIdx.x;
    uint32_t nchunks = (uint32_t)(per / C);
    for (uint32_t k = 0; k < nchunks + S - 1; k++) {
        if (k < nchunks) {
            uint32_t st = k % S;
            if (k >= S) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(C));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su(sm + st * C)),
                         "l"(src + (size_t)k * C), "r"(C), "r"(su(&bar[st])) : "memory");
        }
        if (k >= S - 1) {
            uint32_t j = k - (S - 1), st = j % S;
            asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
                su(&bar[st])), "r"((j / S) & 1));
            for (int f = 0; f < fan; f++)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (size_t)f * bytes + (size_t)j * C),
                             "r"(su(sm + st * C)), "r"(C) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
float timeit(F f, int it = 10) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < it; i++) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / it;
}

int main() {
    const size_t B = (size_t)1 << 30;   // 1 GiB
    char *s, *d; uint32_t *sink;
    cudaMalloc(&s, B); cudaMalloc(&d, 8 * B); cudaMalloc(&sink, 4);
    cudaMemset(s, 1, B);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t n = B / 16;
    for (int grid : {sms * 4, sms * 8, sms * 16}) {
        float t;
        t = timeit([&] { k_write<<<grid, 512>>>((uint4 *)d, n * 4); });
        printf("grid %5d write-only 4 GiB      : %.3f TB/s\n", grid, 4.0 * B / t / 1e9);
        t = timeit([&] { k_read<<<grid, 512>>>((const uint4 *)s, n, sink); });
        printf("grid %5d read-only  1 GiB      : %.3f TB/s\n", grid, 1.0 * B / t / 1e9);
        t = timeit([&] { k_copy<<<grid, 512>>>((uint4 *)d, (const uint4 *)s, n); });
        printf("grid %5d copy LSU   1 GiB      : %.3f TB/s (r+w)\n", grid, 2.0 * B / t / 1e9);
        t = timeit([&] { k_fan8<<<grid, 512>>>((uint4 *)d, (const uint4 *)s, n / 8); });
        printf("grid %5d fan8 LSU 128M->1 GiB  : %.3f TB/s (r+w)\n", grid, 9.0 * B / 8 / t / 1e9);
    }
    auto run_tma = [&](auto kt, int S, int C, const char *tag) {
        cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, S * C);
        for (int cps : {1, 2, 3}) {
            if (S * C * cps > 220 * 1024) continue;
            int grid = sms * cps;
            double done1 = (double)((B / grid) / C) * C * grid;
            double done8 = (double)((B / 8 / grid) / C) * C * grid;
            float t = timeit([&] { kt<<<grid, 32, S * C>>>(d, s, B, 1); });
            printf("%s grid %5d copy TMA   1 GiB      : %.3f TB/s (r+w)\n", tag, grid, 2.0 * done1 / t / 1e9);
            t = timeit([&] { kt<<<grid, 32, S * C>>>(d, s, B / 8, 8); });
            printf("%s grid %5d fan8 TMA 128M->1 GiB  : %.3f TB/s (r+w)\n", tag, grid, 9.0 * done8 / t / 1e9);
        }
    };
    run_tma(k_tma<6, 16384>, 6, 16384, "S6 C16K");
    run_tma(k_tma<4, 32768>, 4, 32768, "S4 C32K");
    run_tma(k_tma<8, 8192>, 8, 8192, "S8 C8K ");
    run_tma(k_tma<3, 65536>, 3, 65536, "S3 C64K");
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}

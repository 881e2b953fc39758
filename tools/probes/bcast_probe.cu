// Probe: the achievable HBM rate of a 1-read : 8-write "broadcast" (the single-GPU allgather's
// traffic pattern: every 16-B vector of an 8 x b source is stored into 8 destination rows), done
// the plainest way -- LSU 16-B loads / stores, grid-stride, full occupancy -- at the sizes where
// the executor's allgather runs below the copy peak.  Prints us per launch (events, 20 launches
// back to back after warm-up) and GB/s of read + write traffic.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void bcast(const uint4 *__restrict__ src, uint4 *__restrict__ dst, uint64_t nv_per_rank, int p) {
    // src: p rows of nv_per_rank vectors; dst: p rows of p * nv_per_rank (row r = concatenation)
    const uint64_t total = (uint64_t)p * nv_per_rank;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(src + i);
        for (int r = 0; r < p; r++) dst[(uint64_t)r * total + i] = v;
    }
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int p = 8;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mib : {1, 2, 4, 8, 16, 64}) {
        const uint64_t b = (uint64_t)mib << 20, nv = b / 16;
        uint4 *s, *d;
        cudaMalloc(&s, p * b);
        cudaMalloc(&d, (uint64_t)p * p * b);
        cudaMemset(s, 1, p * b);
        for (int tpb : {256, 512}) {
            const int grid = sms * (2048 / tpb);
            for (int i = 0; i < 3; i++) bcast<<<grid, tpb>>>(s, d, nv, p);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            for (int i = 0; i < 20; i++) bcast<<<grid, tpb>>>(s, d, nv, p);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / 20, bytes = (double)p * b * (1 + p);
            printf("b=%d MiB tpb=%d: %.1f us  %.0f GB/s (%s)\n", mib, tpb, us, bytes / us / 1e3,
                   cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(s);
        cudaFree(d);
    }
    return 0;
}

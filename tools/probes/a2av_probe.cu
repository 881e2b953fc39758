// Probe: a plain LSU alltoallv for cfg4's shape (p = 8, int64 segments, mean 4 MiB per pair,
// counts uniform on [0, 2 x mean], packed displacements) -- every segment copied with 8-byte
// loads / stores (both sides 8-B aligned; half the segments are not 16-B congruent), grid-
// stride over segments x vectors at full occupancy.  The library's warp-ring executor does the
// same bytes in ~92 us (tools/cfg4_wring.py).  Prints us per launch and GB/s of read + write.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

struct Seg { uint64_t src, dst, n; };   // element offsets (int64) and length

__global__ void a2av(const uint64_t *__restrict__ s, uint64_t *__restrict__ d, const Seg *segs, int nseg,
                     const uint64_t *__restrict__ pre, uint64_t total) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nseg - 1;                       // segment of element i (prefix search)
        while (lo < hi) { int m = (lo + hi + 1) >> 1; if (pre[m] <= i) lo = m; else hi = m - 1; }
        const Seg g = segs[lo];
        const uint64_t k = i - pre[lo];
        d[g.dst + k] = __ldcg(s + g.src + k);
    }
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int p = 8;
    const uint64_t mean_el = (4u << 20) / 8;
    srand(1);
    std::vector<uint64_t> c(p * p);
    for (auto &x : c) x = (uint64_t)(((double)rand() / RAND_MAX) * (2 * mean_el));
    for (int z = 0; z < 6; z++) c[(z * 11) % (p * p)] = 0;
    // packed send rows (rank r's segments for j in order) and recv rows (from j in order)
    std::vector<uint64_t> srow(p, 0), rrow(p, 0);
    for (int r = 0; r < p; r++) for (int j = 0; j < p; j++) { srow[r] += c[r * p + j]; rrow[j] += c[r * p + j]; }
    uint64_t S = 0, R = 0;
    for (int r = 0; r < p; r++) { S = srow[r] > S ? srow[r] : S; R = rrow[r] > R ? rrow[r] : R; }
    std::vector<Seg> segs;
    std::vector<uint64_t> pre;
    uint64_t tot = 0;
    for (int r = 0; r < p; r++) {
        uint64_t so = 0;
        for (int j = 0; j < p; j++) {
            uint64_t ro = 0;
            for (int i = 0; i < r; i++) ro += c[i * p + j];
            segs.push_back(Seg{(uint64_t)r * S + so, (uint64_t)j * R + ro, c[r * p + j]});
            pre.push_back(tot);
            tot += c[r * p + j];
            so += c[r * p + j];
        }
    }
    uint64_t *s, *d, *dpre;
    Seg *dsegs;
    cudaMalloc(&s, p * S * 8); cudaMalloc(&d, p * R * 8);
    cudaMalloc(&dsegs, segs.size() * sizeof(Seg)); cudaMalloc(&dpre, pre.size() * 8);
    cudaMemcpy(dsegs, segs.data(), segs.size() * sizeof(Seg), cudaMemcpyHostToDevice);
    cudaMemcpy(dpre, pre.data(), pre.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(s, 3, p * S * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int tpb : {256, 512}) {
        const int grid = sms * (2048 / tpb);
        for (int i = 0; i < 3; i++) a2av<<<grid, tpb>>>(s, d, dsegs, (int)segs.size(), dpre, tot);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int i = 0; i < 20; i++) a2av<<<grid, tpb>>>(s, d, dsegs, (int)segs.size(), dpre, tot);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / 20;
        printf("tpb=%d: %.1f us, %.0f GB/s (read + write %.1f MB) %s\n", tpb, us, 2.0 * tot * 8 / us / 1e3,
               2.0 * tot * 8 / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

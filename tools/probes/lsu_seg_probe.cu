// Probe: cfg4's alltoallv shape (p = 8, int64 segments, mean 4 MiB per pair, counts uniform on
// [0, 2 x mean], 6 pairs zero, packed displacements) moved by a full-occupancy LSU kernel in
// the style of PyTorch's vectorised copy: every thread owns U consecutive 16-B vectors of
// one segment's destination body (16-B aligned stores) and loads the U (+1 when the source is
// only 8-B congruent) aligned source vectors up front, funnel-shifting them; heads / tails
// (< 16 B per segment end) by one thread per segment, outside the timed launches.  Segment bodies are padded to multiples
// of U vectors in the index space, so a thread's vectors never cross a segment.
// Prints us per launch (20 back-to-back launches) and GB/s of read + write; checks bytes.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

struct Seg {
    uint64_t src, dst, n;      // byte offsets into the send / recv arrays, length
    uint64_t hd;               // head bytes before the 16-B aligned destination body
    uint64_t nv;               // body vectors
    uint64_t v0;               // first padded vector index of this segment
};

__device__ __forceinline__ uint4 shift8(const uint4 &a, const uint4 &b) { return make_uint4(a.z, a.w, b.x, b.y); }

template <int U>
__global__ void __launch_bounds__(256) k_seg(const char *__restrict__ s, char *__restrict__ d, const Seg *__restrict__ segs,
                                             int nseg, uint64_t nvec_pad) {
    for (uint64_t g = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * U; g < nvec_pad;
         g += (uint64_t)gridDim.x * blockDim.x * U) {
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const int m = (lo + hi + 1) >> 1;
            if (segs[m].v0 <= g) lo = m; else hi = m - 1;
        }
        const Seg sg = segs[lo];
        const uint64_t v = g - sg.v0;
        if (v >= sg.nv) continue;
        const int cnt = (int)min((uint64_t)U, sg.nv - v);
        const uint64_t so = sg.src + sg.hd + 16 * v;      // source of this thread's first vector
        uint4 *dv = (uint4 *)(d + sg.dst + sg.hd) + v;
        const uint4 *sv = (const uint4 *)(s + (so & ~15ull));
        if ((so & 15) == 0) {
            uint4 x[U];
#pragma unroll
            for (int k = 0; k < U; k++) if (k < cnt) x[k] = sv[k];
#pragma unroll
            for (int k = 0; k < U; k++) if (k < cnt) dv[k] = x[k];
        } else {   // 8 mod 16 (int64 segments)
            uint4 x[U + 1];
#pragma unroll
            for (int k = 0; k <= U; k++) if (k <= cnt) x[k] = sv[k];
#pragma unroll
            for (int k = 0; k < U; k++) if (k < cnt) dv[k] = shift8(x[k], x[k + 1]);
        }
    }
}
__global__ void k_edges(const char *s, char *d, const Seg *segs, int nseg) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nseg) return;
    const Seg sg = segs[i];
    for (uint64_t b = 0; b < sg.hd && b < sg.n; b++) d[sg.dst + b] = s[sg.src + b];
    for (uint64_t b = sg.hd + 16 * sg.nv; b < sg.n; b++) d[sg.dst + b] = s[sg.src + b];
}

int main(int argc, char **argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int p = 8;
    const uint64_t mean_el = ((argc > 1 ? strtoull(argv[1], 0, 0) : 4ull) << 20) / 8;
    const int elem = argc > 2 ? atoi(argv[2]) : 8;   // 8: int64 segments; 16: 16-B elements (congruent)
    srand(1);
    std::vector<uint64_t> c(p * p);
    for (auto &x : c) x = (uint64_t)(((double)rand() / RAND_MAX) * (2 * mean_el)) * 8 / elem;
    for (int z = 0; z < 6; z++) c[(z * 11) % (p * p)] = 0;
    std::vector<uint64_t> sd(p * p), rd(p * p), srow(p, 0), rrow(p, 0);
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++) { sd[r * p + j] = srow[r]; srow[r] += c[r * p + j]; }
    for (int j = 0; j < p; j++)
        for (int r = 0; r < p; r++) { rd[j * p + r] = rrow[j]; rrow[j] += c[r * p + j]; }
    uint64_t S = 0, R = 0;
    for (int r = 0; r < p; r++) { S = srow[r] > S ? srow[r] : S; R = rrow[r] > R ? rrow[r] : R; }
    const uint64_t Sb = S * elem, Rb = R * elem;
    std::vector<Seg> segs;
    uint64_t v0 = 0, tot = 0;
    const int U = 4;
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++) {
            Seg g;
            g.n = c[r * p + j] * elem;
            if (!g.n) continue;
            g.src = r * Sb + sd[r * p + j] * elem;
            g.dst = j * Rb + rd[j * p + r] * elem;
            g.hd = (16 - (g.dst & 15)) & 15;
            if (g.hd > g.n) g.hd = g.n;
            g.nv = (g.n - g.hd) / 16;
            g.v0 = v0;
            v0 += (g.nv + U - 1) / U * U;
            tot += g.n;
            segs.push_back(g);
        }
    printf("cfg4 shape: mean %llu B, elem %d, %zu segments, %.1f MB moved (read + write %.1f MB)\n",
           (unsigned long long)(mean_el * 8), elem, segs.size(), tot / 1e6, 2 * tot / 1e6);
    char *s, *d;
    Seg *dseg;
    CK(cudaMalloc(&s, p * Sb + 64));
    CK(cudaMalloc(&d, p * Rb + 64));
    CK(cudaMalloc(&dseg, segs.size() * sizeof(Seg)));
    CK(cudaMemcpy(dseg, segs.data(), segs.size() * sizeof(Seg), cudaMemcpyHostToDevice));
    std::vector<unsigned char> h(p * Sb);
    for (uint64_t i = 0; i < h.size(); i++) h[i] = (unsigned char)(i * 131 + (i >> 11));
    CK(cudaMemcpy(s, h.data(), h.size(), cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    for (int bps : {4, 8, 16}) {
        auto go = [&]() {
            k_seg<U><<<nsm * bps, 256>>>(s, d, dseg, (int)segs.size(), v0);
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
        const double us = ms * 1e3 / 20;
        printf("  %d CTAs/SM x 256 threads, %d vectors per thread: %.1f us  %.0f GB/s\n", bps, U, us,
               2.0 * tot / (us * 1e-6) / 1e9);
    }
    k_edges<<<1, 64>>>(s, d, dseg, (int)segs.size());   // (edges once, for the check)
    CK(cudaDeviceSynchronize());
    std::vector<unsigned char> o(p * Rb);
    CK(cudaMemcpy(o.data(), d, o.size(), cudaMemcpyDeviceToHost));
    uint64_t bad = 0;
    for (const Seg &g : segs)
        for (uint64_t b = 0; b < g.n; b++) bad += o[g.dst + b] != h[g.src + b];
    printf("  check: %llu bad bytes\n", (unsigned long long)bad);
    return 0;
}

// Probe: one long copy whose source and destination are 8-B but not 16-B congruent (the
// shape of half of cfg4's int64 alltoallv segments), N bytes, per-warp stage rings of C bytes
// in a grid of 148 CTAs.  Modes:
//   0  reference: source 16-B congruent, TMA bulk load + TMA bulk store (the aligned path)
//   1  cp.async 8-B (LDGSTS) into the stage at the destination's alignment + TMA bulk store
//   2  TMA bulk load of the 16-B aligned source span + two LDS.64 + STG.128 (the library's
//      warp-ring shift store)
//   3  reference: source 16-B congruent, cp.async 16-B (LDGSTS) + TMA bulk store
//   (and a plain 8-B LDG / STG kernel, grid-stride at full occupancy)
// Prints us per launch (20 back-to-back launches, events) and GB/s of read + write.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_load(uint32_t dst, const void *src, uint32_t n, uint32_t mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(n) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(n), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t par) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}"
                 ::"r"(mbar), "r"(par) : "memory");
}
__device__ __forceinline__ void tma_store(void *dst, uint32_t src, uint32_t n) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(n) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// chunk order: 0 = round-robin (chunk gw + i * tw: all warps on one moving front),
// 1 = blocked (warp gw streams chunks [gw * per, (gw + 1) * per): tw independent streams;
// timing only -- the nch % tw tail chunks are skipped, so its byte check reports them)
__constant__ int c_blocked;
__device__ __forceinline__ uint64_t chunk_of(uint64_t gw, uint64_t i, uint64_t tw, uint64_t nch) {
    return c_blocked ? gw * (nch / tw) + i : gw + i * tw;
}
// chunk C, stages per warp S, loads in flight D, warps per CTA W
// mode 0 / 2: per-warp ring, lane 0 loads D ahead through mbarriers
template <int MODE, int C, int S, int D, int W>
__global__ void __launch_bounds__(W * 32) k_tma(const char *src, char *dst, uint64_t nch) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t mb[W][S];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    char *st = sm + (size_t)w * S * (C + 16);
    if (l == 0) for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t tw = (uint64_t)gridDim.x * W, gw = (uint64_t)blockIdx.x * W + w;
    const uint64_t n_mine = c_blocked ? nch / tw : (gw < nch ? (nch - gw + tw - 1) / tw : 0);
    const uint32_t lb = MODE == 0 ? C : C + 16;
    auto issue = [&](uint64_t i) {
        const uint64_t k = chunk_of(gw, i, tw, nch);
        const char *a = MODE == 0 ? src + k * C : (const char *)(((uintptr_t)(src + k * C)) & ~(uintptr_t)15);
        tma_load(su32(st + (i % S) * (C + 16)), a, lb, su32(&mb[w][i % S]));
    };
    if (l == 0) for (uint64_t i = 0; i < (uint64_t)D && i < n_mine; i++) issue(i);
    for (uint64_t i = 0; i < n_mine; i++) {
        const uint64_t k = chunk_of(gw, i, tw, nch);
        char *stg = st + (i % S) * (C + 16);
        mbar_wait(su32(&mb[w][i % S]), (uint32_t)((i / S) & 1));
        if (MODE == 0) {
            if (l == 0) tma_store(dst + k * C, su32(stg), C);
        } else {
            const char *b = stg + 8;   // payload byte 0 (source is 8 mod 16)
            for (int j = l; j < C / 16; j += 32) {
                const uint2 lo = *reinterpret_cast<const uint2 *>(b + 16 * j);
                const uint2 hi = *reinterpret_cast<const uint2 *>(b + 16 * j + 8);
                *reinterpret_cast<uint4 *>(dst + k * C + 16 * j) = make_uint4(lo.x, lo.y, hi.x, hi.y);
            }
        }
        __syncwarp();
        if (l == 0 && i + D < n_mine) {
            if (MODE == 0 && i + D >= (uint64_t)S) wait_read<S - D - 1>();   // stage (i+D)%S's store done reading
            issue(i + D);
        }
    }
    if (MODE == 0 && l == 0) wait_all();
}

__device__ __forceinline__ void cpa8(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// mode 1: cp.async 8-B into the stage, lane 0 bulk-stores D chunks behind
template <int C, int S, int D, int W, int V = 8>
__global__ void __launch_bounds__(W * 32) k_cpa(const char *src, char *dst, uint64_t nch) {
    extern __shared__ __align__(128) char sm[];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    char *st = sm + (size_t)w * S * C;
    const uint64_t tw = (uint64_t)gridDim.x * W, gw = (uint64_t)blockIdx.x * W + w;
    const uint64_t n_mine = c_blocked ? nch / tw : (gw < nch ? (nch - gw + tw - 1) / tw : 0);
    auto flush = [&](uint64_t i) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (l == 0) tma_store(dst + chunk_of(gw, i, tw, nch) * C, su32(st + (i % S) * C), C);
    };
    for (uint64_t i = 0; i < n_mine; i++) {
        if (i >= (uint64_t)S) {          // stage i%S: chunk i-S's store must have read it
            if (l == 0) wait_read<S - D - 1>();
            __syncwarp();
        }
        const char *a = src + chunk_of(gw, i, tw, nch) * C;
        const uint32_t s0 = su32(st + (i % S) * C);
        if (V == 8) {
            for (int j = l; j < C / 8; j += 32) cpa8(s0 + 8 * j, a + 8 * j);
        } else {
            for (int j = l; j < C / 16; j += 32) cpa16(s0 + 16 * j, a + 16 * j);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (i >= (uint64_t)D) {
            asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory");
            flush(i - D);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (uint64_t i = n_mine > (uint64_t)D ? n_mine - D : 0; i < n_mine; i++) flush(i);
    if (l == 0) wait_all();
}

__global__ void k_lsu(const uint64_t *src, uint64_t *dst, uint64_t n8) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n8; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = __ldcg(src + i);
}

char *src, *dst;
cudaEvent_t e0, e1;

template <int C, int S, int D, int W, int B>
void run(uint64_t N, bool check) {
    const uint64_t nch = N / C;
    const size_t sm0 = (size_t)W * S * (C + 16), sm1 = (size_t)W * S * C;
    if (B * sm0 > 220 * 1024) { printf("C=%d S=%d D=%d W=%d B=%d: smem too large\n", C, S, D, W, B); return; }
    CK(cudaFuncSetAttribute(k_tma<0, C, S, D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0));
    CK(cudaFuncSetAttribute(k_tma<2, C, S, D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0));
    CK(cudaFuncSetAttribute(k_cpa<C, S, D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    CK(cudaFuncSetAttribute(k_cpa<C, S, D, W, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    printf("C=%d S=%d D=%d W=%d CTAs/SM=%d N=%llu MiB:", C, S, D, W, B, (unsigned long long)(N >> 20));
    for (int mode = 0; mode < 4; mode++) {
        auto go = [&]() {
            if (mode == 3) k_cpa<C, S, D, W, 16><<<148 * B, W * 32, sm1>>>(src, dst, nch);
            if (mode == 0) k_tma<0, C, S, D, W><<<148 * B, W * 32, sm0>>>(src, dst, nch);
            if (mode == 1) k_cpa<C, S, D, W><<<148 * B, W * 32, sm1>>>(src + 8, dst, nch);
            if (mode == 2) k_tma<2, C, S, D, W><<<148 * B, W * 32, sm0>>>(src + 8, dst, nch);
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
        printf("  m%d %.1f us %.0f GB/s", mode, us, 2.0 * N / (us * 1e-6) / 1e9);
    }
    printf("\n");
    if (!check) return;
    unsigned char *h = (unsigned char *)malloc(N + 64), *g = (unsigned char *)malloc(N);
    for (uint64_t i = 0; i < N + 64; i++) h[i] = (unsigned char)(i * 131 + (i >> 12));
    CK(cudaMemcpy(src, h, N + 64, cudaMemcpyHostToDevice));
    for (int mode = 1; mode <= 2; mode++) {
        CK(cudaMemset(dst, 0, N));
        if (mode == 1) k_cpa<C, S, D, W><<<148 * B, W * 32, sm1>>>(src + 8, dst, nch);
        else k_tma<2, C, S, D, W><<<148 * B, W * 32, sm0>>>(src + 8, dst, nch);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(g, dst, N, cudaMemcpyDeviceToHost));
        uint64_t bad = 0;
        for (uint64_t i = 0; i < N; i++) bad += g[i] != h[i + 8];
        printf("  mode %d check: %llu bad bytes\n", mode, (unsigned long long)bad);
    }
    free(h); free(g);
}

int main(int argc, char **argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const uint64_t N = (argc > 1 ? strtoull(argv[1], 0, 0) : 256ull) << 20;
    const int blocked = argc > 2 ? atoi(argv[2]) : 0;
    CK(cudaMemcpyToSymbol(c_blocked, &blocked, sizeof blocked));
    printf("# chunk order: %s\n", blocked ? "blocked (one stream per warp)" : "round-robin (one moving front)");
    CK(cudaMalloc(&src, N + 64));
    CK(cudaMalloc(&dst, N + 64));
    CK(cudaMemset(src, 1, N + 64));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    {   // plain LSU reference
        for (int i = 0; i < 3; i++) k_lsu<<<148 * 4, 512>>>((const uint64_t *)(src + 8), (uint64_t *)dst, N / 8);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int i = 0; i < 20; i++) k_lsu<<<148 * 4, 512>>>((const uint64_t *)(src + 8), (uint64_t *)dst, N / 8);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("lsu 8-B N=%llu MiB: %.1f us %.0f GB/s\n", (unsigned long long)(N >> 20), ms * 1e3 / 20, 2.0 * N / (ms * 1e-3 / 20) / 1e9);
    }
    run<4096, 6, 3, 8, 1>(N, true);     // the library's warp rings (4 warps x 2 CTAs / SM)
    run<4096, 6, 4, 4, 2>(N, false);
    run<16384, 6, 4, 1, 2>(N, false);   // the library's producer ring shape (one ring per CTA)
    run<8192, 6, 4, 2, 2>(N, false);
    run<4096, 12, 8, 2, 2>(N, false);
    run<4096, 6, 4, 1, 4>(N, false);
    run<8192, 6, 4, 1, 4>(N, false);
    run<32768, 6, 4, 1, 1>(N, false);
    return 0;
}

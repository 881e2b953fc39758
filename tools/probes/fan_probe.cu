// Probe: does the ORDER of a TMA fan-out's stores matter for the single-GPU allgather's
// 1-read : p-write traffic?  One producer thread per CTA (2 CTAs / SM, 296 CTAs, like the
// library's dynamic executor) takes groups of G x C bytes of the p x b source from a work
// queue, TMA-loads the group into one half of a double-buffered 2 x 48 KiB shared-memory
// ring, and stores it to the p destination rows:
//   order 0 (chunk-major, the library's): for each chunk, p bulk stores of C bytes;
//   order 1 (destination-major): for each destination, the G chunks (G*C contiguous bytes);
//   order 2 (destination-major, one op): one bulk store of G*C bytes per destination.
// Also a write-only reference (order 3: the same stores without any load).  Prints us per
// launch (20 launches back to back) and TB/s of read + write traffic, per b and order.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 2) fan(const char *src, char *dst, uint64_t b, int p, uint32_t C, int G,
                                              int order, int split, unsigned *queue, unsigned *done) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t mbar[2];
    const uint64_t total = (uint64_t)p * b;        // source bytes
    const uint64_t grp = (uint64_t)G * C;
    const uint32_t ngroups = (uint32_t)((total + grp - 1) / grp);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        uint32_t ph[2] = {0, 0};
        int k = 0;
        for (uint32_t u = atomicAdd(queue, 1u); u < ngroups; u = atomicAdd(queue, 1u), k ^= 1) {
            const uint64_t off = (uint64_t)u * grp;
            const uint32_t n = (uint32_t)(off + grp <= total ? grp : total - off);
            char *buf = sm + k * 49152;
            // the half's previous stores have read shared memory (one group committed per use)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            if (order != 3) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar[k])), "r"(n)
                             : "memory");
                const uint32_t lc = split ? C : n;   // split: one load op per C-byte chunk
                for (uint32_t c = 0; c < n; c += lc)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(su32(buf + c)), "l"(src + off + c), "r"(n - c < lc ? n - c : lc), "r"(su32(&mbar[k]))
                                 : "memory");
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                                 "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(su32(&mbar[k])), "r"(ph[k]) : "memory");
                ph[k] ^= 1;
            }
            // destination row r: dst + r * total + off (allgather: row r = concatenation)
            if (order == 0) {
                for (uint32_t c = 0; c < n; c += C) {
                    const uint32_t len = n - c < C ? n - c : C;
                    for (int r = 0; r < p; r++)
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                     ::"l"(dst + (uint64_t)r * total + off + c), "r"(su32(buf + c)), "r"(len) : "memory");
                }
            } else if (order == 1) {
                for (int r = 0; r < p; r++)
                    for (uint32_t c = 0; c < n; c += C) {
                        const uint32_t len = n - c < C ? n - c : C;
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                     ::"l"(dst + (uint64_t)r * total + off + c), "r"(su32(buf + c)), "r"(len) : "memory");
                    }
            } else {
                for (int r = 0; r < p; r++)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                 ::"l"(dst + (uint64_t)r * total + off), "r"(su32(buf)), "r"(n) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        // last CTA resets the queue (graph / back-to-back launches)
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) { *queue = 0; *done = 0; }
    }
}


// The library's producer shape: a ring of NS stages of C bytes, loads kept AHEAD chunks in
// front of the oldest pending store, pieces of PC chunks from the work queue, chunk-major
// fan-out stores (one bulk group per chunk).
__global__ void __launch_bounds__(128, 2) ring(const char *src, char *dst, uint64_t b, int p, uint32_t C, int NS,
                                               int AHEAD, int PC, unsigned *queue, unsigned *done) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t mbar[8];
    __shared__ uint64_t soff[8];
    __shared__ uint32_t slen[8];
    const uint64_t total = (uint64_t)p * b;
    const uint64_t piece = (uint64_t)PC * C;
    const uint32_t npieces = (uint32_t)((total + piece - 1) / piece);
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        uint32_t issued = 0, stored = 0;
        auto store_one = [&]() {
            const uint32_t s = stored % NS;
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(su32(&mbar[s])), "r"((stored / NS) & 1u) : "memory");
            for (int r = 0; r < p; r++)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(dst + (uint64_t)r * total + soff[s]), "r"(su32(sm + (size_t)s * C)), "r"(slen[s]) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            stored++;
        };
        for (uint32_t u = atomicAdd(queue, 1u); u < npieces; u = atomicAdd(queue, 1u)) {
            const uint64_t p0 = (uint64_t)u * piece, p1 = p0 + piece < total ? p0 + piece : total;
            for (uint64_t off = p0; off < p1; off += C) {
                const uint32_t n = (uint32_t)(p1 - off < C ? p1 - off : C);
                if (issued - stored == (uint32_t)AHEAD) store_one();
                const uint32_t s = issued % NS;
                if (issued >= (uint32_t)NS) {
                    const int w = (int)(stored - 1 - (issued - NS));
                    if (w <= 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    else if (w == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    else if (w == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
                    else if (w == 3) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
                }
                soff[s] = off;
                slen[s] = n;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar[s])), "r"(n) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(sm + (size_t)s * C)), "l"(src + off), "r"(n), "r"(su32(&mbar[s])) : "memory");
                issued++;
            }
        }
        while (stored < issued) store_one();
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) { *queue = 0; *done = 0; }
    }
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int p = 8;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(fan, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
    unsigned *q;
    cudaMalloc(&q, 64);
    cudaMemset(q, 0, 64);
    const int grid = 2 * sms;
    struct Shape { uint32_t C; int G; } shapes[] = {{16384, 3}, {8192, 6}, {49152, 1}};
    for (int mib : {4, 8, 64}) {
        const uint64_t b = (uint64_t)mib << 20;
        char *s, *d;
        cudaMalloc(&s, p * b);
        cudaMalloc(&d, (uint64_t)p * p * b);
        cudaMemset(s, 1, p * b);
        for (const Shape &sh : shapes) {
            for (int oi = 0; oi < 5; oi++) {
                const int order = oi == 4 ? 0 : oi, split = oi == 4;
                if (sh.G == 1 && (order == 1 || split)) continue;
                for (int i = 0; i < 3; i++) fan<<<grid, 128, 98304>>>(s, d, b, p, sh.C, sh.G, order, split, q, q + 1);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                for (int i = 0; i < 20; i++) fan<<<grid, 128, 98304>>>(s, d, b, p, sh.C, sh.G, order, split, q, q + 1);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const double us = ms * 1e3 / 20, bytes = (double)p * b * (order == 3 ? p : 1 + p);
                printf("b=%2d MiB C=%5u G=%d order=%d split=%d: %8.2f us  %.3f TB/s (%s)\n", mib, sh.C, sh.G, order, split, us,
                       bytes / us / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
        cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
        struct RS { uint32_t C; int NS, AHEAD, PC; } rs[] = {{16384, 6, 4, 1}, {16384, 6, 4, 3}, {16384, 6, 2, 1},
                                                               {16384, 6, 5, 1}, {8192, 8, 6, 2}, {32768, 3, 2, 1}};
        for (const RS &r : rs) {
            for (int i = 0; i < 3; i++) ring<<<grid, 128, 98304>>>(s, d, b, p, r.C, r.NS, r.AHEAD, r.PC, q, q + 1);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            for (int i = 0; i < 20; i++) ring<<<grid, 128, 98304>>>(s, d, b, p, r.C, r.NS, r.AHEAD, r.PC, q, q + 1);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / 20, bytes = (double)p * b * (1 + p);
            printf("b=%2d MiB ring C=%5u NS=%d AHEAD=%d PC=%d: %8.2f us  %.3f TB/s (%s)\n", mib, r.C, r.NS, r.AHEAD, r.PC,
                   us, bytes / us / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(s);
        cudaFree(d);
    }
    return 0;
}

// Auxiliary sm_100a kernels of libmpxa: the A2 counts exchange + exclusive scans
// (mpxa_counts_kernel, mpxa_scan_kernel) and the f3 partitioned point-to-point kernels (cycle
// starts, host-enqueued Pready -- LSU or TMA slices --, stream-ordered Parrived / completion),
// with their host launchers.
#include "kern_common.cuh"

namespace mpxa {

// ------------------------------------------------------------------------------------
// A2: counts exchange + exclusive scan, all ranks on this device (single-process mode).
//   recvcounts[r*p + j] = sendcounts[j*p + r];  rdispls[r*p + j] = sum_{i<j} recvcounts[r*p+i]
// One warp per receiving rank r, 32 entries per iteration, carry across iterations.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int64_t warp_incl_scan(int64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

__global__ void mpxa_counts_kernel(const int64_t *__restrict__ sendcounts, int64_t *__restrict__ recvcounts,
                                   int64_t *__restrict__ rdispls, int p, int r0, int nr) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= nr) return;
    int r = r0 + warp;                  // global receiving rank
    int64_t carry = 0;
    for (int j0 = 0; j0 < p; j0 += 32) {
        int j = j0 + lane;
        int64_t v = j < p ? sendcounts[(int64_t)j * p + r] : 0;
        int64_t inc = warp_incl_scan(v, lane);
        if (j < p) {
            recvcounts[(int64_t)warp * p + j] = v;
            rdispls[(int64_t)warp * p + j] = carry + inc - v;
        }
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
}

// exclusive scan of nr rows of p entries (rows already gathered into `counts`)
__global__ void mpxa_scan_kernel(const int64_t *__restrict__ counts, int64_t *__restrict__ recvcounts,
                                 int64_t *__restrict__ rdispls, int p, int nr) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= nr) return;
    int64_t carry = 0;
    for (int j0 = 0; j0 < p; j0 += 32) {
        int j = j0 + lane;
        int64_t v = j < p ? counts[(int64_t)warp * p + j] : 0;
        int64_t inc = warp_incl_scan(v, lane);
        if (j < p) {
            recvcounts[(int64_t)warp * p + j] = v;
            rdispls[(int64_t)warp * p + j] = carry + inc - v;
        }
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
}

// ------------------------------------------------------------------------------------
// f3: partitioned point-to-point.  Cycle counters and flags live in the
// comm's partition heap; the sender's partitions go straight into the receiver's buffer.
// ------------------------------------------------------------------------------------
// (all partitioned kernels are PDL launches: they wait for the preceding kernel's completion
// before touching anything, then let the next launch start its own prologue)
__device__ __forceinline__ void part_enter() {
    griddep_wait();
    griddep_launch_dependents();
}

__global__ void part_start_send(unsigned long long *scycle) {
    part_enter();
    if (threadIdx.x == 0) *scycle += 1ull;
}

// receiver enters the next cycle: everything stream-ordered before it (its consumers of the
// previous cycle) is done, so the sender may overwrite the buffer -> clear-to-send
__global__ void part_start_recv(unsigned long long *rcycle, unsigned long long *cts_remote) {
    part_enter();
    if (threadIdx.x == 0) {
        const unsigned long long c = *rcycle + 1ull;
        *rcycle = c;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(cts_remote), "l"(c) : "memory");
    }
}

// host-enqueued Pready of sender partitions [p0, p0 + gridDim.x / nct): nct CTAs per partition
__global__ void __launch_bounds__(256) part_pready(mpxa_psend_dev_t ch, int p0, unsigned long long chunk,
                                                   unsigned int nct) {
    part_enter();
    const int i = p0 + (int)(blockIdx.x / nct);
    const unsigned long long k = blockIdx.x % nct;
    const unsigned long long lo = k * chunk;
    const unsigned long long hi = lo + chunk < ch.part_bytes ? lo + chunk : ch.part_bytes;
    mpxa_dev_pready_part(&ch, i, lo, hi, nct);
}

// Host-enqueued Pready of large 16-B aligned partitions: the same (partition, slice) CTAs, each
// slice streamed by ONE thread through a TMA ring (kPartStages x kPartChunk of shared memory,
// loads kept kPartAhead chunks ahead of the oldest store) instead of the CTA's LSU loop (4 x 16 B
// in flight per thread): f3 256 MiB in 16 partitions, see DESIGN §8 f3.  The slice's bulk
// writes complete (wait_group 0) and are fenced to the generic proxy before the CTA counts
// itself (acq_rel) and the last CTA of the partition releases its arrival flag.
constexpr int kPartStages = 4, kPartAhead = 3;
constexpr unsigned long long kPartTmaMin = 64ull << 20;   // calls from 64 MiB take the TMA slices (measured:
                                                         // the LSU loop is as fast or faster below)
constexpr unsigned long long kPartSliceMax = 256ull << 10;
constexpr uint32_t kPartChunk = 16384;
__global__ void __launch_bounds__(32) part_pready_tma(mpxa_psend_dev_t ch, int p0, unsigned long long chunk,
                                                      unsigned int nct) {
    extern __shared__ __align__(128) char pbuf[];
    __shared__ __align__(8) uint64_t mbar[kPartStages];
    const int i = p0 + (int)(blockIdx.x / nct);
    const unsigned long long k = blockIdx.x % nct;
    const unsigned long long lo = k * chunk;
    const unsigned long long hi = lo + chunk < ch.part_bytes ? lo + chunk : ch.part_bytes;
    // the slice's first chunks into L2 before the dependency wait -- a cache fill only, read
    // after the wait (measured, 256 MiB cycle 98.6-100.1 -> 97.3-98.8 us)
    if (threadIdx.x == 0 && hi > lo)
        prefetch_l2((uintptr_t)(ch.src + (unsigned long long)i * ch.part_bytes + lo),
                    (uint32_t)min(hi - lo, (unsigned long long)kPartAhead * kPartChunk));
    part_enter();
    if (threadIdx.x != 0) return;
    const unsigned long long cyc = *(volatile const unsigned long long *)ch.scycle;
    if (mpxa_dev_wait_ge(ch.cts, cyc, ch.err, ch.timeout_ns)) return;   // clear to send
    for (int s = 0; s < kPartStages; s++) mbar_init(smem_u32(&mbar[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const char *src = (const char *)ch.src + (unsigned long long)i * ch.part_bytes;
    char *dst = (char *)ch.dst + (unsigned long long)i * ch.part_bytes;
    uint32_t issued = 0, stored = 0;
    __shared__ unsigned long long ooff[kPartStages];   // each stage's offset / length
    __shared__ uint32_t olen[kPartStages];
    auto store_one = [&]() {
        const uint32_t st = stored % kPartStages;
        mbar_wait(smem_u32(&mbar[st]), (stored / kPartStages) & 1u);
        tma_store_1d(dst + ooff[st], smem_u32(pbuf + (size_t)st * kPartChunk), olen[st]);
        bulk_commit();
        stored++;
    };
    for (unsigned long long o = lo; o < hi; o += kPartChunk) {
        if (issued - stored == (uint32_t)kPartAhead) store_one();
        const uint32_t st = issued % kPartStages;
        if (issued >= (uint32_t)kPartStages) bulk_wait_read((int)(stored - 1 - (issued - kPartStages)));
        ooff[st] = o;
        olen[st] = (uint32_t)(hi - o < kPartChunk ? hi - o : kPartChunk);
        tma_load_1d(smem_u32(pbuf + (size_t)st * kPartChunk), src + o, olen[st], smem_u32(&mbar[st]));
        issued++;
    }
    while (stored < issued) store_one();
    bulk_wait_all();
    fence_proxy_async();   // the bulk writes before the generic-proxy release below
    unsigned int prev = 0u;
    if (nct > 1u) asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&ch.done[i]) : "memory");
    if (prev + 1u == nct) {
        if (nct > 1u) ch.done[i] = 0;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&ch.arr[i]), "l"(cyc) : "memory");
    }
}

// stream-ordered Parrived / completion: block until flags[lo, hi) >= *cycle (one CTA)
__global__ void part_wait_flags(const unsigned long long *flags, int lo, int hi, const unsigned long long *cycle,
                                int *err, long long timeout_ns) {
    part_enter();
    __shared__ unsigned long long want;
    if (threadIdx.x == 0) want = *(volatile const unsigned long long *)cycle;
    __syncthreads();
    for (int i = lo + (int)threadIdx.x; i < hi; i += blockDim.x) {
        unsigned long long t0 = 0;
        int it = 0;
        while (mpxa_dev_ld_acquire(flags + i) < want) {
            if (++it > 32) {
                __nanosleep(256);
                if (!t0) t0 = mpxa_dev_now();
                else if ((long long)(mpxa_dev_now() - t0) > timeout_ns) { atomicExch(err, 1); break; }
            }
        }
    }
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

cudaError_t launch_part_start(bool sender, unsigned long long *cycle, unsigned long long *cts_remote,
                              cudaStream_t stream) {
    if (sender) return launch_pdl(part_start_send, dim3(1), dim3(32), stream, cycle);
    return launch_pdl(part_start_recv, dim3(1), dim3(32), stream, cycle, cts_remote);
}

cudaError_t launch_part_pready(const mpxa_psend_dev_t &ch, int p0, int np, cudaStream_t stream) {
    // large 16-B aligned calls: TMA slices, 3 CTAs per SM (64 KiB of shared memory each),
    // slices a multiple of 16 B
    if (np > 0 && ch.part_bytes * (unsigned long long)np >= kPartTmaMin &&
        !(((uintptr_t)ch.src | (uintptr_t)ch.dst | ch.part_bytes) & 15)) {
        static cudaError_t a = cudaFuncSetAttribute(part_pready_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)(kPartStages * kPartChunk));
        if (a != cudaSuccess) return a;
        // slices: the call's bytes over one wave of 3 CTAs / SM, at most kPartSliceMax -- large
        // calls run several waves of short slices, so SMs that stream faster take more of them
        // (the block scheduler balances; one wave of long slices waits for the slowest SMs:
        // measured, 256 MiB in 16 partitions 107 -> 99.7 us per cycle, 128-256 KiB slices best)
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
        unsigned long long nct = 3ull * (unsigned long long)sms / (unsigned long long)np;   // one wave
        if (nct < 1) nct = 1;
        unsigned long long per = ((ch.part_bytes + nct - 1) / nct + 15) & ~15ull;
        if (per > kPartSliceMax) per = kPartSliceMax;   // large calls: several waves of short slices
        if (per < kPartChunk) per = kPartChunk;
        nct = (ch.part_bytes + per - 1) / per;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(np * nct));
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = kPartStages * kPartChunk;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, part_pready_tma, ch, p0, per, (unsigned)nct);
    }
    // CTAs per partition: 32 KiB pieces, up to ~4 waves of the machine over the whole call
    const unsigned long long chunk = 32ull << 10;
    unsigned long long nct = (ch.part_bytes + chunk - 1) / chunk;
    const unsigned long long cap = np > 0 ? (4ull * 148 + np - 1) / np : 1;
    if (nct > cap) nct = cap;
    if (nct < 1) nct = 1;
    const unsigned long long per = (ch.part_bytes + nct - 1) / nct;
    const unsigned long long ch16 = (per + 15) & ~15ull;
    nct = ch16 ? (ch.part_bytes + ch16 - 1) / ch16 : 1;
    if (nct < 1) nct = 1;
    return launch_pdl(part_pready, dim3((unsigned)(np * nct)), dim3(256), stream, ch, p0,
                      (unsigned long long)(ch16 ? ch16 : 1), (unsigned)nct);
}

cudaError_t launch_part_wait(const unsigned long long *flags, int lo, int hi, const unsigned long long *cycle,
                             int *err, long long timeout_ns, cudaStream_t stream) {
    return launch_pdl(part_wait_flags, dim3(1), dim3(256), stream, flags, lo, hi, cycle, err, timeout_ns);
}

cudaError_t launch_counts(const int64_t *sc, int64_t *rc, int64_t *rd, int p, int r0, int nr,
                          cudaStream_t stream) {
    int threads = 256, warps_per = threads / 32;
    int blocks = (nr + warps_per - 1) / warps_per;
    if (blocks < 1) blocks = 1;
    mpxa_counts_kernel<<<blocks, threads, 0, stream>>>(sc, rc, rd, p, r0, nr);
    return cudaGetLastError();
}

cudaError_t launch_scan(const int64_t *counts, int64_t *rc, int64_t *rd, int p, int nr,
                        cudaStream_t stream) {
    int threads = 256, warps_per = threads / 32;
    int blocks = (nr + warps_per - 1) / warps_per;
    if (blocks < 1) blocks = 1;
    mpxa_scan_kernel<<<blocks, threads, 0, stream>>>(counts, rc, rd, p, nr);
    return cudaGetLastError();
}

}  // namespace mpxa

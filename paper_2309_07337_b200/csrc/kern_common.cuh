// Device primitives and helpers shared by the sm_100a kernels of libmpxa (exec_kernel.cu,
// small_kernels.cu, aux_kernels.cu): system- / GPU-scope acquire-release
// flags, PDL, 16-B vector loads / stores, LSU copy loops, TMA bulk copies (cp.async.bulk,
// SASS UBLKCP) with mbarriers, column slices, and register-staged 16-byte pieces.
// Payloads are opaque bytes: only integer vector loads/stores, never a float conversion.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpxa_internal.h"
#include "../../include/mpxa_device.cuh"

namespace mpxa {

// ------------------------------------------------------------------------------------
// memory primitives
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Signalling pattern: every thread's data stores, __syncthreads, then one thread's release
// store at system scope.  The release is cumulative over everything that happens-before it
// (the CTA barrier orders the other threads' stores before it; the producer's bulk stores
// are completed and proxy-fenced before the barrier), so no separate fence.sc.sys is issued:
// it compiled to MEMBAR.SC.SYS + L1 invalidation and cost ~2-4 us per signal (clock64
// stamps, 4 emulated GPUs).
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// GPU-scope counters (row barriers, launch completion): release / acq_rel RMWs instead of
// __threadfence() (fence.sc.gpu) + a relaxed atomic -- the same cumulative ordering
__device__ __forceinline__ void red_release_gpu_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_acq_rel_gpu_add(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// Programmatic dependent launch (launches carry programmaticStreamSerialization): the
// prologue (program tables: library-owned, immutable while launches are in flight) overlaps
// the previous kernel's tail; everything that kernel may have written or still reads (user
// buffers, workspace, epoch, flags) is touched only after griddepcontrol.wait, which returns
// once the preceding grid has completed and its memory is visible.  No-op without PDL.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Source loads are cache-global (.cg: L2 only, never an L1 line).  RECV / WORK may have been
// written earlier in the same launch by another SM or a peer GPU; SEND is read-only inside
// the launch, but under PDL the launch began before its producer finished, so no source is
// read through the non-coherent path either.  (RO is kept as the call sites' statement of
// which buffers are read-only.)
template <bool RO>
__device__ __forceinline__ uint4 ld16(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st16(uint4 *p, const uint4 &v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w) : "memory");
}
template <typename T>
__device__ __forceinline__ T ldcg(const T *p) { return __ldcg(p); }
template <>
__device__ __forceinline__ uint8_t ldcg<uint8_t>(const uint8_t *p) {
    unsigned short v;
    asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return (uint8_t)v;
}

// LSU copies.  Deliberately NOT templated on width / thread count / unroll: the executor
// must stay small enough for the instruction cache (a template-expanded version was 87 K
// SASS instructions and spent small launches stalled on instruction fetch).
//
// Copy n bytes with nt cooperating threads (index t).  The SOURCE side is always read in
// 16-byte aligned vectors, kLsuUnroll of them in flight per thread (loads are what bound an
// LSU copy's bandwidth: stores are fire-and-forget); each vector is stored in pieces of the
// widest access class W the destination allows at that offset ((dst - src) mod 16).  Bytes
// before the first aligned source vector and after the last are copied singly.
#ifndef MPXA_LSU_UNROLL
#define MPXA_LSU_UNROLL 8
#endif
constexpr int kLsuUnroll = MPXA_LSU_UNROLL;

__device__ __forceinline__ void store_w(char *d, const uint4 &v, unsigned W) {
    switch (W) {
        case 16: st16((uint4 *)d, v); break;
        case 8:
            ((uint2 *)d)[0] = make_uint2(v.x, v.y);
            ((uint2 *)d)[1] = make_uint2(v.z, v.w);
            break;
        case 4: {
            uint32_t *q = (uint32_t *)d;
            q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
            break;
        }
        default: {
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            if (W == 2) {
#pragma unroll
                for (int i = 0; i < 8; i++) ((uint16_t *)d)[i] = (uint16_t)(w[i >> 1] >> (16 * (i & 1)));
            } else {
#pragma unroll
                for (int i = 0; i < 16; i++) d[i] = (char)(w[i >> 2] >> (8 * (i & 3)));
            }
        }
    }
}

static __device__ __noinline__ void lsu_copy_range(char *dst, const char *src, uint64_t n, int t, int nt, bool ro) {
    (void)ro;
    if (n == 0) return;
    uint64_t head = (16 - ((uintptr_t)src & 15)) & 15;
    if (head > n) head = n;
    for (uint64_t i = t; i < head; i += nt) dst[i] = (char)ldcg((const uint8_t *)src + i);
    const uint64_t nv = (n - head) >> 4;
    const uint4 *s4 = (const uint4 *)(src + head);
    char *d = dst + head;
    const unsigned m = (unsigned)((uintptr_t)d & 15);
    const unsigned W = m == 0 ? 16u : (m & -m);
    // shifted full-vector stores pay off once every warp has a whole block of spans
    for (uint64_t i0 = t; i0 < nv; i0 += (uint64_t)kLsuUnroll * nt) {
        uint4 v[kLsuUnroll];
#pragma unroll
        for (int k = 0; k < kLsuUnroll; k++) {
            const uint64_t i = i0 + (uint64_t)k * nt;
            if (i < nv) v[k] = ld16<false>(s4 + i);
        }
#pragma unroll
        for (int k = 0; k < kLsuUnroll; k++) {
            const uint64_t i = i0 + (uint64_t)k * nt;
            if (i < nv) store_w(d + 16 * i, v[k], W);
        }
    }
    for (uint64_t k = head + nv * 16 + t; k < n; k += nt) dst[k] = (char)ldcg((const uint8_t *)src + k);
}

// Fan-out: one read, nd stores, when every destination shares the source's 16-B alignment.
static __device__ __noinline__ void lsu_copy_fan(char *const *dsts, int nd, const char *src, uint64_t n, int t, int nt,
                                          bool ro) {
    if (n == 0) return;
    unsigned mis = 0;
    for (int k = 0; k < nd; k++) mis |= (unsigned)(((uintptr_t)dsts[k] ^ (uintptr_t)src) & 15);
    if (mis) {
        for (int k = 0; k < nd; k++) lsu_copy_range(dsts[k], src, n, t, nt, ro);
        return;
    }
    uint64_t head = (16 - ((uintptr_t)src & 15)) & 15;
    if (head > n) head = n;
    for (uint64_t i = t; i < head; i += nt) {
        const char b = (char)ldcg((const uint8_t *)src + i);
        for (int k = 0; k < nd; k++) dsts[k][i] = b;
    }
    const uint4 *s4 = (const uint4 *)(src + head);
    const uint64_t nv = (n - head) >> 4;
    for (uint64_t i = t; i < nv; i += nt) {
        const uint4 v = ro ? ld16<true>(s4 + i) : ld16<false>(s4 + i);
        for (int k = 0; k < nd; k++) st16((uint4 *)(dsts[k] + head) + i, v);
    }
    for (uint64_t k2 = head + nv * 16 + t; k2 < n; k2 += nt) {
        const char b = (char)ldcg((const uint8_t *)src + k2);
        for (int k = 0; k < nd; k++) dsts[k][k2] = b;
    }
}

// ------------------------------------------------------------------------------------
// executor
// ------------------------------------------------------------------------------------
constexpr uint64_t kLine = 128;          // slice boundaries are 128-B multiples of a move
constexpr uint64_t kTmaMin = 2048;       // aligned slices at least this long go through TMA
constexpr uint64_t kLsuBig = 8192;       // misaligned slices at least this long use all LSU warps
constexpr int kWarps = kThreads / 32;
constexpr int kLsuWarps = kWarps - 1;    // warp 0 is the TMA producer
constexpr int kLsuThreads = kThreads - 32;

// ---- TMA bulk copies (cp.async.bulk: SASS UBLKCP) --------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_load_1d(uint32_t dst_smem, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst_smem), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n}" ::"r"(mbar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_store_1d(void *dst, uint32_t src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read(int n) {
    switch (n) {
        case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.bulk.wait_group.read 5;" ::: "memory"); break;
        case 6: asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory"); break;
        case 7: asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory"); break;
        default: asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory"); break;
    }
}
// bulk prefetch of [a, a + bytes) into L2 (16-B aligned, a 16-B multiple)
__device__ __forceinline__ void prefetch_l2(uintptr_t a, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

__device__ __forceinline__ int clampi(int64_t v, int n) { return v < 0 ? 0 : v > n ? n : (int)v; }

__device__ __forceinline__ void slice_of(uint64_t nbytes, int c, int nC, uint64_t &lo, uint64_t &hi) {
    uint64_t nl = (nbytes + kLine - 1) / kLine;
    lo = ((uint64_t)c * nl / nC) * kLine;
    hi = ((uint64_t)(c + 1) * nl / nC) * kLine;
    if (hi > nbytes) hi = nbytes;
    if (lo > hi) lo = hi;
}

#ifdef MPXA_TRACE
// phase stamps of CTA 0 in SM cycles (clock64: one SM, so comparable and cycle-accurate)
#define TRACE(k) do { if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x == 0 || threadIdx.x == 32)) P.dc->trace[(k) + (threadIdx.x ? 16 : 0)] = (uint64_t)clock64(); } while (0)
#ifdef MPXA_CTA_TRACE_OWNER
__device__ uint64_t g_cta_trace[6][kMaxCtas];   // per-CTA entry / exit / after the dependency wait / first piece / classified / first store (GPU 0)
#define CTA_STAMP(w) do { if (threadIdx.x == 0 && blockIdx.y == 0) g_cta_trace[w][blockIdx.x] = globaltimer(); } while (0)
#else
#define CTA_STAMP(w) do { } while (0)
#endif
#else
#define TRACE(k) do { } while (0)
#define CTA_STAMP(w) do { } while (0)
#endif

// a step as one CTA sees it (executor and small-kernel step tables in shared memory)
struct StepInfo {
    int32_t first;          // index of this CTA's first move (flow group range start)
    int32_t nm;             // number of moves in this CTA's flow group range
    uint32_t signal_mask, wait_mask;
};

// store_piece with generic stores only (the destination may be shared memory)
__device__ __forceinline__ void store_piece_generic(char *dp, uint4 v, uint32_t len) {
    if (len == 16 && (((uintptr_t)dp) & 15) == 0) { *(uint4 *)dp = v; return; }
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if ((len & 3) == 0 && (((uintptr_t)dp) & 3) == 0) {
        uint32_t *d = (uint32_t *)dp;
        for (uint32_t b = 0; b < len / 4; b++) d[b] = w[b];
        return;
    }
    for (uint32_t b = 0; b < len; b++) dp[b] = (char)(w[b >> 2] >> (8 * (b & 3)));
}

// Batched copy of up to kBatch SMALL moves by one warp (n <= 512 B each): every lane loads
// its 16-byte piece of every move first (kBatch loads in flight), then stores them -- one
// memory round trip per batch instead of one per move.  Byte-granular when a piece is not
// 16-B aligned on both sides.
#ifndef MPXA_KBATCH
#define MPXA_KBATCH 4
#endif
constexpr int kBatch = MPXA_KBATCH;
constexpr uint64_t kSmallMax = 512;

// Up to 16 bytes at any alignment, in registers: the (at most five) aligned words that
// overlap [sp, sp+len) are loaded independently (one round trip), then funnel-shifted.
// Only words holding wanted bytes are touched, so nothing outside the 4-byte granules of
// the piece is read.
// A batch of up to kBatch 16-byte pieces: every load of the batch is issued before any
// loaded register is touched (a use right after a load -- even a register move where two
// code paths merge -- would expose one memory latency per piece).  A16: every piece is a
// whole, 16-B aligned 16-byte vector on both sides (one LDG.128 / STG.128 each); otherwise
// the aligned words overlapping each piece are loaded and funnel-shifted at store time.
struct PieceRef {
    const char *src;
    uint32_t len;     // 0: no piece
};
// AW: 16 -- the host vouched that every piece is a whole, 16-B aligned vector; 8 -- every
// offset, length, base and stride is a multiple of 8 (int64 / double payloads): pieces move as
// 8-byte words; 0 -- any alignment: aligned 4-byte words and funnel shifts
template <int AW>
struct PieceRegs {
    uint4 v[kBatch];
    uint32_t w4[kBatch];
    __device__ __forceinline__ void issue(int k, const char *sp, uint32_t len) {
        if (AW == 16) {
            v[k] = ld16<false>((const uint4 *)sp);
        } else if (AW == 8) {
            const uint2 lo = __ldcg((const uint2 *)sp);
            const uint2 hi = len > 8 ? __ldcg((const uint2 *)sp + 1) : make_uint2(0u, 0u);
            v[k] = make_uint4(lo.x, lo.y, hi.x, hi.y);
        } else if (AW == 4) {   // 4-B aligned, len a multiple of 4: whole words, no shifts
            const uint32_t *wp = (const uint32_t *)sp;
            v[k].x = __ldcg(wp);
            v[k].y = len > 4 ? __ldcg(wp + 1) : 0u;
            v[k].z = len > 8 ? __ldcg(wp + 2) : 0u;
            v[k].w = len > 12 ? __ldcg(wp + 3) : 0u;
        } else {
            const uintptr_t a = (uintptr_t)sp & ~(uintptr_t)3;
            const uint32_t *wp = (const uint32_t *)a;
            const uintptr_t end = (uintptr_t)sp + len;
            v[k].x = __ldcg(wp);                        // a < end always (len >= 1)
            v[k].y = (a + 4 < end) ? __ldcg(wp + 1) : 0u;
            v[k].z = (a + 8 < end) ? __ldcg(wp + 2) : 0u;
            v[k].w = (a + 12 < end) ? __ldcg(wp + 3) : 0u;
            w4[k] = (a + 16 < end) ? __ldcg(wp + 4) : 0u;
        }
    }
    // the same with generic loads (the source may be shared memory)
    __device__ __forceinline__ void issue_generic(int k, const char *sp, uint32_t len) {
        if (AW == 16) { v[k] = *(const uint4 *)sp; return; }
        if (AW == 8) {
            const uint2 lo = *(const uint2 *)sp;
            const uint2 hi = len > 8 ? *((const uint2 *)sp + 1) : make_uint2(0u, 0u);
            v[k] = make_uint4(lo.x, lo.y, hi.x, hi.y);
            return;
        }
        const uintptr_t a = (uintptr_t)sp & ~(uintptr_t)3;
        const uint32_t *wp = (const uint32_t *)a;
        const uintptr_t end = (uintptr_t)sp + len;
        v[k].x = wp[0];
        v[k].y = (a + 4 < end) ? wp[1] : 0u;
        v[k].z = (a + 8 < end) ? wp[2] : 0u;
        v[k].w = (a + 12 < end) ? wp[3] : 0u;
        w4[k] = (a + 16 < end) ? wp[4] : 0u;
    }
    __device__ __forceinline__ uint4 value(int k, const char *sp) const {
        if (AW != 0) return v[k];
        const uint32_t sh = 8u * (uint32_t)((uintptr_t)sp & 3);
        return make_uint4(__funnelshift_r(v[k].x, v[k].y, sh), __funnelshift_r(v[k].y, v[k].z, sh),
                          __funnelshift_r(v[k].z, v[k].w, sh), __funnelshift_r(v[k].w, w4[k], sh));
    }
};

// AW as in PieceRegs
template <int AW = 0>
__device__ __forceinline__ void store_piece(char *dp, uint4 v, uint32_t len) {
    if (AW == 16 || (len == 16 && (((uintptr_t)dp) & 15) == 0)) { st16((uint4 *)dp, v); return; }
    if (AW == 8) {                                      // 8-B aligned, len 8 or 16
        *(uint2 *)dp = make_uint2(v.x, v.y);
        if (len > 8) *((uint2 *)dp + 1) = make_uint2(v.z, v.w);
        return;
    }
    if (AW == 4) {                                      // 4-B aligned, len 4, 8, 12 or 16
        uint32_t *d = (uint32_t *)dp;
        d[0] = v.x;
        if (len > 4) d[1] = v.y;
        if (len > 8) d[2] = v.z;
        if (len > 12) d[3] = v.w;
        return;
    }
    if (len == 16 && (((uintptr_t)dp) & 3) == 0) {
        uint32_t *d = (uint32_t *)dp;
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
        return;
    }
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if ((len & 3) == 0 && (((uintptr_t)dp) & 3) == 0) {   // whole 4-byte words (e.g. 4-B elements)
        uint32_t *d = (uint32_t *)dp;
        d[0] = v.x;
        if (len > 4) d[1] = v.y;
        if (len > 8) d[2] = v.z;
        return;
    }
    for (uint32_t b = 0; b < len; b++) dp[b] = (char)(w[b >> 2] >> (8 * (b & 3)));
}

// Launch with the PDL attribute (pdl) and/or cooperatively.  cooperative = 1: the grid's CTAs
// wait on one another (emulated GPUs' CTA rows, per-step row barriers, peers across processes)
// and must be co-resident -- a cooperative launch guarantees it; 2: the same with PDL as well
// (accepted on sm_100a: tools/probes/coop_probe.cu, +0.1-0.25 us per launch over PDL alone).
// A cooperative launch the device cannot make co-resident falls back to the plain launch
// (grids are sized to the co-resident count, so this is a guard, not a path).
static inline cudaError_t launch_kernel(void (*kern)(ExecParams), const ExecParams &P, dim3 grid, dim3 block, size_t smem,
                                 int cooperative, bool pdl, cudaStream_t stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (cooperative) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        na++;
    }
    if (!cooperative || cooperative == 2) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        na++;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P);
    if (e == cudaErrorCooperativeLaunchTooLarge && cooperative == 2) {
        (void)cudaGetLastError();
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, P);
    }
    return e;
}

}  // namespace mpxa

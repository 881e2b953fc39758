// sm_100a kernels of the mpxa hot path.
//
//  mpxa_exec_kernel   -- executes a collective PROGRAM (mpxa_internal.h): every step of
//                        pairwise / Bruck / ring / hierarchical alltoall(v) and allgather
//                        (SURVEY.md §8(a) A3-A8).  Column-slice ownership: CTA c moves
//                        slice c of every move, so steps are separated by __syncthreads
//                        only; cross-GPU dependencies use per-(src GPU, CTA) release/acquire
//                        flags plus one clear-to-send (CTS) flag per GPU pair (A9).
//  mpxa_counts_kernel -- counts exchange + exclusive scan (A2) for ranks resident on this
//                        device, one warp per receiving rank, __shfl_up_sync scans.
//  mpxa_scan_kernel   -- exclusive scan only (multi-process path: counts arrive through
//                        an exchange program first).
//
// Payloads are opaque bytes: only integer vector loads/stores, never a float conversion.
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

__device__ __noinline__ void lsu_copy_range(char *dst, const char *src, uint64_t n, int t, int nt, bool ro) {
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
__device__ __noinline__ void lsu_copy_fan(char *const *dsts, int nd, const char *src, uint64_t n, int t, int nt,
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
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

__device__ __forceinline__ int clampi(int64_t v, int n) { return v < 0 ? 0 : v > n ? n : (int)v; }

__device__ __forceinline__ void slice_of(uint64_t nbytes, int c, int nC, uint64_t &lo, uint64_t &hi) {
    uint64_t nl = (nbytes + kLine - 1) / kLine;
    lo = ((uint64_t)c * nl / nC) * kLine;
    hi = ((uint64_t)(c + 1) * nl / nC) * kLine;
    if (hi > nbytes) hi = nbytes;
    if (lo > hi) lo = hi;
}

struct RingEntry {
    char *dst;          // non-fanout destination of the chunk
    uint64_t doff;      // fanout: byte offset inside every rank's dst_kind buffer
    uint32_t len;
    uint8_t fanout, dst_kind;
};

#ifdef MPXA_TRACE
__device__ uint64_t g_cta_trace[6][kMaxCtas];   // per-CTA entry / exit / after the dependency wait / first piece / classified / first store (GPU 0)
#define CTA_STAMP(w) do { if (threadIdx.x == 0 && blockIdx.y == 0) g_cta_trace[w][blockIdx.x] = globaltimer(); } while (0)
// phase stamps of CTA 0 in SM cycles (clock64: one SM, so comparable and cycle-accurate)
#define TRACE(k) do { if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x == 0 || threadIdx.x == 32)) P.dc->trace[(k) + (threadIdx.x ? 16 : 0)] = (uint64_t)clock64(); } while (0)
#else
#define TRACE(k) do { } while (0)
#define CTA_STAMP(w) do { } while (0)
#endif
static_assert(kMoveTile <= kThreads, "prologue prefetch: one move per thread");
struct StepInfo {
    int32_t first;          // index of this CTA's first move (flow group range start)
    int32_t nm;             // number of moves in this CTA's flow group range
    uint32_t signal_mask, wait_mask;
};

struct ExecShared {
    char *recv_base[kMaxGpus];
    char *work_base[kMaxGpus];
    SymRegion *sym[kMaxGpus];
    Move moves[kMoveTile];
    uint64_t mbar[kMaxStages];
    RingEntry ring[kMaxStages];
    StepInfo steps[kMaxStepsSmem];   // this CTA's view of every step, loaded once
    uint64_t epoch;      // this launch's epoch (device-side sequence number)
    uint32_t cts_ok;     // remote GPUs whose CTS for this epoch was observed
    uint32_t kuni0;      // dynamic mode: dyn_classify's result for step 0's first tile when classified
                         // in the prologue (before the dependency wait)
    int abort_flag;
    uint32_t pcA[kMoveTile + 1];  // dynamic mode: exclusive prefix of TMA pieces per move
    uint32_t pcB[kMoveTile + 1];  //               and of LSU pieces per move
    const char *msrc[kMoveTile];  //               resolved source of each move
    uint64_t mdst[kMoveTile];     //               destination address (fan-out: offset)
    uint64_t wsum[kThreads / 32];
    // warp-ring mode: per-warp stage barriers and the descriptor of each stage's contents
    uint64_t wmbar[kWarpsExec][kWStages];
    struct WEntry {
        const char *src;    // kind 0: 16-B aligned body source; kind 1: payload source
        char *dst;          // kind 0 non-fanout / kind 1: destination
        uint64_t doff;      // kind 0 fan-out: offset inside every rank's dst_kind buffer
        uint32_t n;         // payload bytes
        uint32_t lbytes;    // bytes loaded into the stage (16-B multiple)
        uint16_t sh;        // kind 1: payload byte 0 sits at stage + sh
        uint8_t kind;       // 0: bulk-store stage; 1: warp stores shifted out of the stage
        uint8_t fanout, dst_kind;
    } went[kWarpsExec][kWStages];
    uint32_t wseq[kWarpsExec];   // loads issued on each warp's ring so far in this launch (stage
                                 // index and mbarrier phase continue across tiles and steps)
};

__device__ __forceinline__ char *base_of(const ExecParams &P, const ExecShared &S, int kind, int rank) {
    int g = rank / P.R;
    uint64_t local = (uint64_t)(rank - g * P.R);
    if (kind == BK_SEND)   // sources are always local: only this process's (or virtual GPU's) ranks
        return (char *)P.send + (P.mode == 2 ? 0 : (uint64_t)g * P.R * P.send_stride) + local * P.send_stride;
    if (kind == BK_RECV) return S.recv_base[g] + local * P.recv_stride;
    return S.work_base[g] + local * P.work_stride;
}

// Fan-out bulk store of one staged chunk to offset doff of the dst_kind buffer of every rank:
// the ranks' bases walked GPU by GPU (no per-rank division, unlike base_of).
__device__ __forceinline__ void fan_store(const ExecParams &P, const ExecShared &S, int kind, uint64_t doff,
                                          uint32_t src, uint32_t len) {
    const uint64_t stride = kind == BK_RECV ? P.recv_stride : P.work_stride;
    for (int g = 0; g < P.G; g++) {
        char *b = (kind == BK_RECV ? S.recv_base[g] : S.work_base[g]) + doff;
        for (int l = 0; l < P.R; l++, b += stride) tma_store_1d(b, src, len);
    }
}

// Spin (threads < 32, one per bit of mask) until *slot(bit) >= want; sets abort on timeout.
#ifndef MPXA_POLL_NS
#define MPXA_POLL_NS 128   // executor flag polls: back-off between system-scope loads
#endif
__device__ __noinline__ void wait_mask_ge(const ExecParams &P, ExecShared &S, uint32_t mask,
                                             const uint64_t *slot0, uint64_t stride_elems,
                                             uint64_t want) {
    int t = threadIdx.x;
    if (t < 32 && ((mask >> t) & 1u)) {
        const uint64_t *slot = slot0 + (uint64_t)t * stride_elems;
        uint64_t start = 0;
        int it = 0;
        while (ld_acquire_sys(slot) < want) {
            if (++it > 32) {
                __nanosleep(MPXA_POLL_NS);
                if (start == 0) start = globaltimer();
                else if ((int64_t)(globaltimer() - start) > P.timeout_ns) {
                    atomicExch(P.err, 1);
                    S.abort_flag = 1;
                    break;
                }
            }
            if (*(volatile int *)&S.abort_flag) break;
        }
    }
}

// The single-thread TMA producer: a ring of kRingStages smem stages (= P.stages, a compile-time
// constant so the ring index is a multiply, not a division); loads run P.ahead chunks
// ahead of the oldest pending store; each chunk's stores form one bulk group.
struct Producer {
    uint32_t issued = 0, stored = 0;
    char *stages;

    __device__ __forceinline__ void store_one(const ExecParams &P, ExecShared &S) {
        const uint32_t s = stored % kRingStages;
        mbar_wait(smem_u32(&S.mbar[s]), (stored / kRingStages) & 1u);
        const RingEntry e = S.ring[s];
#ifdef MPXA_TRACE
        if (stored == 0) CTA_STAMP(5);
#endif
        const uint32_t src = smem_u32(stages + (size_t)s * P.chunk);
        if (!e.fanout) {
            tma_store_1d(e.dst, src, e.len);
        } else {
            fan_store(P, S, e.dst_kind, e.doff, src, e.len);
        }
        bulk_commit();
        stored++;
    }
    __device__ __forceinline__ void push(const ExecParams &P, ExecShared &S, const char *src, const RingEntry &e) {
        if (issued - stored == (uint32_t)P.ahead) store_one(P, S);
        const uint32_t ns = kRingStages;
        const uint32_t s = issued % ns;
        if (issued >= ns) bulk_wait_read((int)(stored - 1 - (issued - ns)));
        S.ring[s] = e;
        tma_load_1d(smem_u32(stages + (size_t)s * P.chunk), src, e.len, smem_u32(&S.mbar[s]));
        issued++;
    }
    __device__ __forceinline__ void drain(const ExecParams &P, ExecShared &S, bool consumed) {
        while (stored < issued) store_one(P, S);
        if (consumed) {
            bulk_wait_all();
            fence_proxy_async();   // bulk writes before generic readers / flag release
        } else {
            // nothing in this launch reads the data again: only the shared-memory source
            // must outlive the CTA (kernel completion publishes the global writes)
            bulk_wait_read(0);
        }
    }
};

// How CTA (flow group f, slice sl) handles one move: byte range of its slice, source and
// destination addresses, and the path (TMA body + LSU head/tail, or LSU only).
struct MovePlan {
    const char *src;
    char *dst;          // non-fanout
    uint64_t doff;      // offset inside each rank's dst buffer (fanout)
    uint64_t n;         // slice bytes
    bool tma;
    uint32_t head;      // TMA: bytes before the 16-B aligned body
    uint64_t body;      // TMA: aligned body bytes (multiple of 16)
};

// Slice bounds of a move length, cached per thread: uniform ops have one length for every
// move, so the 64-bit divisions run once per launch instead of once per move.
struct SliceCache {
    uint64_t len = ~0ull, lo = 0, hi = 0;
    __device__ __forceinline__ void get(uint64_t nbytes, int sl, int nS, uint64_t &l, uint64_t &h) {
        if (nbytes != len) {
            len = nbytes;
            slice_of(nbytes, sl, nS, lo, hi);
        }
        l = lo;
        h = hi;
    }
};

__device__ __noinline__ unsigned fan_misalign(const ExecParams &P, const ExecShared &S, int kind, uint64_t doff,
                                              const char *src) {
    unsigned mis = 0;
    for (int j = 0; j < P.p; j++) mis |= (unsigned)(((uintptr_t)(base_of(P, S, kind, j) + doff) ^ (uintptr_t)src) & 15);
    return mis;
}

// slice length only (cheap classification shared by every thread)
__device__ __forceinline__ uint64_t slice_len(const ExecParams &P, const Move &m, int sl, SliceCache &sc,
                                              uint64_t &lo) {
    uint64_t hi;
    sc.get((uint64_t)m.len * P.unit, sl, P.nS, lo, hi);
    return hi - lo;
}

__device__ __forceinline__ MovePlan plan_move(const ExecParams &P, const ExecShared &S, const Move &m, int sl, SliceCache &sc) {
    MovePlan mp;
    uint64_t lo;
    mp.n = slice_len(P, m, sl, sc, lo);
    mp.src = base_of(P, S, m.src_kind, m.src_rank) + (uint64_t)m.src_off * P.unit + lo;
    mp.doff = (uint64_t)m.dst_off * P.unit + lo;
    mp.dst = m.fanout ? nullptr : base_of(P, S, m.dst_kind, m.dst_rank) + mp.doff;
    const unsigned mis = !m.fanout ? (unsigned)(((uintptr_t)mp.dst ^ (uintptr_t)mp.src) & 15)
                                   : fan_misalign(P, S, m.dst_kind, mp.doff, mp.src);
    mp.tma = mis == 0 && mp.n >= kTmaMin;
    mp.head = (uint32_t)((16 - ((uintptr_t)mp.src & 15)) & 15);
    if (mp.head > mp.n) mp.head = (uint32_t)mp.n;
    mp.body = (mp.n - mp.head) & ~(uint64_t)15;
    return mp;
}

__device__ __noinline__ void lsu_copy(const ExecParams &P, const ExecShared &S, const Move &m, const MovePlan &mp,
                                         uint64_t off, uint64_t n, int t, int nt) {
    const bool ro = m.src_kind == BK_SEND;
    if (!m.fanout) {
        lsu_copy_range(mp.dst + off, mp.src + off, n, t, nt, ro);
    } else {
        char *dsts[8];
        for (int j0 = 0; j0 < P.p; j0 += 8) {
            const int nd = min(8, P.p - j0);
            for (int k = 0; k < nd; k++) dsts[k] = base_of(P, S, m.dst_kind, j0 + k) + mp.doff + off;
            lsu_copy_fan(dsts, nd, mp.src + off, n, t, nt, ro);
        }
    }
}

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

struct SmallJob {
    const char *src;
    char *dst;          // non-fanout destination (or first fan-out destination offset base)
    uint64_t doff;
    uint32_t n;
    uint8_t fanout, dst_kind, ro;
};

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

// Batched copy of up to kBatch SMALL moves by one warp (n <= 512 B each): lane l moves bytes
// [16l, 16l+16) of every move; all loads of the batch are issued before any store.
template <bool A16>
__device__ __forceinline__ void small_batch_t(const ExecParams &P, const ExecShared &S, const SmallJob *jobs, int nj,
                                              int lane) {
    PieceRegs<A16 ? 16 : 0> R;
    const uint32_t o = (uint32_t)lane * 16;
#pragma unroll
    for (int k = 0; k < kBatch; k++)
        if (k < nj && o < jobs[k].n) R.issue(k, jobs[k].src + o, min(16u, jobs[k].n - o));
    TRACE(7);
#pragma unroll
    for (int k = 0; k < kBatch; k++) {
        if (k >= nj || o >= jobs[k].n) continue;
        const SmallJob &j = jobs[k];
        const uint32_t len = min(16u, j.n - o);
        const uint4 val = R.value(k, j.src + o);
        if (!j.fanout) {
            store_piece(j.dst + o, val, len);
        } else {
            for (int r = 0; r < P.p; r++) store_piece(base_of(P, S, j.dst_kind, r) + j.doff + o, val, len);
        }
    }
}

__device__ __noinline__ void small_batch(const ExecParams &P, const ExecShared &S, const SmallJob *jobs, int nj,
                                            int lane) {
    TRACE(6);
    // every piece whole and 16-B aligned on both sides (uniform across the warp)?
    bool a16 = true;
    for (int k = 0; k < nj; k++) {
        const SmallJob &j = jobs[k];
        uintptr_t bits = (uintptr_t)j.src | (uintptr_t)j.n;
        if (!j.fanout) bits |= (uintptr_t)j.dst;
        else
            for (int r = 0; r < P.p; r++) bits |= (uintptr_t)(base_of(P, S, j.dst_kind, r) + j.doff);
        a16 = a16 && (bits & 15) == 0;
    }
    if (a16) small_batch_t<true>(P, S, jobs, nj, lane);
    else small_batch_t<false>(P, S, jobs, nj, lane);
    TRACE(8);
}

// Dynamic mode (ExecParams::dyn_units != 0; single-step programs): the step's moves (all in
// S.moves) are cut into pieces of at most dyn_u bytes, taken from device work queues until
// they run dry (per-SM bandwidth differs across the chip, so static slices leave a tail of
// slow CTAs).  Moves whose source and destination(s) are 16-B congruent feed queue A: the
// producer thread streams those pieces through the TMA ring (bytes outside the aligned
// body copied by that thread).  All other moves feed queue B: each LSU warp takes pieces on
// its own and copies them with 16-B source vectors and destination-width stores.  The
// queues are independent, so neither role waits for the other.  Returns whether this
// thread issued generic stores.
// Up to 15 bytes [o, o+n) of a piece whose source and destination(s) are 16-B congruent:
// split into naturally aligned 1/2/4/8-byte accesses, every load issued before any store.
__device__ __noinline__ void copy_edge(const ExecParams &P, const ExecShared &S, const Move &m, const MovePlan &mp,
                                       uint64_t o, uint32_t n) {
    uint64_t v[7];
    uint8_t sz[7];
    int k = 0;
    const char *a = mp.src + o;
    for (uint32_t done = 0; done < n && k < 7; k++) {
        const uintptr_t x = (uintptr_t)(a + done);
        uint32_t w = 8;
        while (w > 1 && ((x & (w - 1)) || w > n - done)) w >>= 1;
        sz[k] = (uint8_t)w;
        const char *q = a + done;
        v[k] = w == 8 ? __ldcg((const unsigned long long *)q)
             : w == 4 ? __ldcg((const unsigned int *)q)
             : w == 2 ? __ldcg((const unsigned short *)q) : (uint64_t)ldcg((const uint8_t *)q);
        done += w;
    }
    const int nd = m.fanout ? P.p : 1;
    for (int j = 0; j < nd; j++) {
        char *d = (m.fanout ? base_of(P, S, m.dst_kind, j) + mp.doff : mp.dst) + o;
        uint32_t done = 0;
        for (int i = 0; i < k; i++) {
            char *q = d + done;
            switch (sz[i]) {
                case 8: *(unsigned long long *)q = v[i]; break;
                case 4: *(unsigned int *)q = (unsigned int)v[i]; break;
                case 2: *(unsigned short *)q = (unsigned short)v[i]; break;
                default: *q = (char)v[i];
            }
            done += sz[i];
        }
    }
}

__device__ __forceinline__ int find_move(const uint32_t *pc, int nm, uint32_t u) {
    int lo = 0, hi = nm - 1;      // last move with pc[m] <= u (moves with no piece are skipped)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pc[mid] <= u) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ MovePlan piece_plan(const ExecParams &P, const ExecShared &S, int mi, uint64_t lo,
                                               uint64_t U) {
    const Move &m = S.moves[mi];
    MovePlan mp;
    const uint64_t L = (uint64_t)m.len * P.unit;
    mp.src = S.msrc[mi] + lo;
    mp.doff = (m.fanout ? S.mdst[mi] : 0) + lo;
    mp.dst = m.fanout ? nullptr : (char *)(uintptr_t)S.mdst[mi] + lo;
    mp.n = min(L, lo + U) - lo;
    return mp;
}

// Load (unless prefetched) and classify one tile of moves: S.msrc / S.mdst resolved, and the
// exclusive piece prefixes S.pcA (16-B congruent moves of >= kTmaMin bytes: the TMA queue)
// and S.pcB (the rest), totals at index nm.
// Returns k > 0 when every move of the tile is in the TMA queue with the same number k of
// pieces (uniform alltoall / allgather blocks): piece u is then piece u % k of move u / k, no
// search of the prefix array.
__device__ __noinline__ uint32_t dyn_classify(const ExecParams &P, ExecShared &S, int g, int first, int nm,
                                              bool loaded) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint64_t U = (uint64_t)P.dyn_u;
    if (!loaded) {   // moves not prefetched by the prologue (later tiles, or step 0 not dense)
        __syncthreads();   // everyone is done with the previous tile's moves
        if (t < nm) S.moves[t] = P.mode == 1 ? P.progs[g].moves[first + t] : P.prog.moves[first + t];
        __syncthreads();
    }
    // classify each move (one per thread: nm <= kMoveTile = kThreads) and count its pieces;
    // one 64-bit block scan gives both prefixes (A in the low, B in the high half)
    uint64_t kt = 0;
    if (t < nm) {
        const Move &m = S.moves[t];
        const uint64_t L = (uint64_t)m.len * P.unit;
        const char *src = base_of(P, S, m.src_kind, m.src_rank) + (uint64_t)m.src_off * P.unit;
        const uint64_t doff = (uint64_t)m.dst_off * P.unit;
        char *dst = m.fanout ? nullptr : base_of(P, S, m.dst_kind, m.dst_rank) + doff;
        S.msrc[t] = src;
        S.mdst[t] = m.fanout ? doff : (uint64_t)(uintptr_t)dst;
        const unsigned mis = !m.fanout ? (unsigned)(((uintptr_t)dst ^ (uintptr_t)src) & 15)
                                       : fan_misalign(P, S, m.dst_kind, doff, src);
        const uint64_t k = (L + U - 1) / U;
        kt = (mis == 0 && L >= kTmaMin) ? k : (k << 32);
    }
    uint64_t inc = kt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) S.wsum[warp] = inc;
    __syncthreads();
    uint64_t wo = 0;
    for (int w = 0; w < warp; w++) wo += S.wsum[w];
    const uint64_t ex = wo + inc - kt;
    S.pcA[t] = (uint32_t)ex;
    S.pcB[t] = (uint32_t)(ex >> 32);
    if (t == kThreads - 1) {
        S.pcA[kThreads] = (uint32_t)(wo + inc);
        S.pcB[kThreads] = (uint32_t)((wo + inc) >> 32);
    }
    __syncthreads();
    const uint32_t k0 = S.pcA[1];
    const int uni = __syncthreads_and(t >= nm || (kt == (uint64_t)k0 && k0 > 0));
    return uni ? k0 : 0u;
}

// One tile of at most kMoveTile moves (queues of tile ti).
__device__ __noinline__ bool dyn_tile(const ExecParams &P, ExecShared &S, Producer &prod, int g, int first, int nm,
                                      bool loaded, bool classified, int ti) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint64_t U = (uint64_t)P.dyn_u, chunk = (uint64_t)P.chunk;
    const uint32_t kuni = classified ? S.kuni0 : dyn_classify(P, S, g, first, nm, loaded);
    CTA_STAMP(4);
    const uint32_t totA = S.pcA[nm], totB = S.pcB[nm];
    bool wrote = false;
    if (t == 0) {
        if (totA == 0) return false;
        uint32_t *q = &P.dc->dyn_next[g * kMaxDynTiles + ti];
        uint32_t u = atomicAdd(q, 1u);
        CTA_STAMP(3);
        while (u < totA) {
            const uint32_t un = atomicAdd(q, 1u);   // next piece requested while this one streams
            const int mi = kuni ? (int)(u / kuni) : find_move(S.pcA, nm, u);
            const Move &m = S.moves[mi];
            const MovePlan mp = piece_plan(P, S, mi, (uint64_t)(u - S.pcA[mi]) * U, U);
            const uint64_t nb = mp.n;
            uint64_t head = (16 - ((uintptr_t)mp.src & 15)) & 15;
            if (head > nb) head = nb;
            const uint64_t body = (nb - head) & ~(uint64_t)15;
            // head and tail bytes (< 16 each; congruent piece: widest aligned accesses)
            if (head) { copy_edge(P, S, m, mp, 0, (uint32_t)head); wrote = true; }
            if (nb > head + body) { copy_edge(P, S, m, mp, head + body, (uint32_t)(nb - head - body)); wrote = true; }
            for (uint64_t o = 0; o < body; o += chunk) {
                RingEntry e;
                e.len = (uint32_t)min(chunk, body - o);
                e.fanout = m.fanout;
                e.dst_kind = m.dst_kind;
                e.doff = mp.doff + head + o;
                e.dst = m.fanout ? nullptr : mp.dst + head + o;
                prod.push(P, S, mp.src + head + o, e);
            }
            u = un;
        }
    } else if (warp >= 1 && totB) {
        uint32_t *q = &P.dc->dyn_next2[g * kMaxDynTiles + ti];
        uint32_t un = 0;
        if (lane == 0) un = atomicAdd(q, 1u);
        for (;;) {
            const uint32_t u = __shfl_sync(0xffffffffu, un, 0);
            if (u >= totB) break;
            if (lane == 0) un = atomicAdd(q, 1u);   // next piece requested while this one copies
            const int mi = find_move(S.pcB, nm, u);
            const Move &m = S.moves[mi];
            const MovePlan mp = piece_plan(P, S, mi, (uint64_t)(u - S.pcB[mi]) * U, U);
            lsu_copy(P, S, m, mp, 0, mp.n, lane, 32);
            wrote = true;
        }
    }
    return wrote;
}

// 16 bytes starting at byte d (0..15) of the 32-byte pair (a, b)
__device__ __forceinline__ uint4 shift16(const uint4 &a, const uint4 &b, uint32_t d) {
    uint32_t x0, x1, x2, x3, x4;
    switch (d >> 2) {
        case 0: x0 = a.x; x1 = a.y; x2 = a.z; x3 = a.w; x4 = b.x; break;
        case 1: x0 = a.y; x1 = a.z; x2 = a.w; x3 = b.x; x4 = b.y; break;
        case 2: x0 = a.z; x1 = a.w; x2 = b.x; x3 = b.y; x4 = b.z; break;
        default: x0 = a.w; x1 = b.x; x2 = b.y; x3 = b.z; x4 = b.w; break;
    }
    const uint32_t r = 8u * (d & 3u);
    if (!r) return make_uint4(x0, x1, x2, x3);
    return make_uint4(__funnelshift_r(x0, x1, r), __funnelshift_r(x1, x2, r), __funnelshift_r(x2, x3, r),
                      __funnelshift_r(x3, x4, r));
}

// 16 bytes starting at byte D of the 32-byte pair (a, b), D a compile-time constant
template <uint32_t D>
__device__ __forceinline__ uint4 shift16c(const uint4 &a, const uint4 &b) {
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    constexpr uint32_t q = D >> 2, r = 8u * (D & 3u);
    if (r == 0) return make_uint4(w[q], w[q + 1], w[q + 2], w[q + 3]);
    return make_uint4(__funnelshift_r(w[q], w[q + 1], r), __funnelshift_r(w[q + 1], w[q + 2], r),
                      __funnelshift_r(w[q + 2], w[q + 3], r), __funnelshift_r(w[q + 3], w[q + 4], r));
}
template <uint32_t D>
__device__ __forceinline__ void shift_loop(const uint4 *s4, uint4 *d4, uint32_t nv, int lane) {
    for (uint32_t v = lane; v < nv; v += 32) st16(d4 + v, shift16c<D>(s4[v], s4[v + 1]));
}

// The warp stores n payload bytes that sit at stage byte sh to dst: 16-B stores at the
// destination's alignment, each assembled from two aligned 16-B shared-memory loads.
__device__ __forceinline__ void wring_shift_store(const char *stage, uint32_t sh, char *dst, uint32_t n, int lane) {
    uint32_t hd = (uint32_t)((16 - ((uintptr_t)dst & 15)) & 15);
    if (hd > n) hd = n;
    for (uint32_t i = lane; i < hd; i += 32) dst[i] = stage[sh + i];
    const uint32_t nv = (n - hd) >> 4;
    const uint32_t o0 = sh + hd, d = o0 & 15;
    const uint4 *s4 = (const uint4 *)(stage + (o0 & ~15u));
    uint4 *d4 = (uint4 *)(dst + hd);
    if (d == 0) {
        for (uint32_t v = lane; v < nv; v += 32) st16(d4 + v, s4[v]);
    } else if (d == 8) {
        // 8-byte elements (the common misalignment): two 8-B shared loads, no shifts (measured,
        // cfg4 int64 mean 4 / 8 MiB: 94.5 / 179.4 -> 89.4 / 166.8 us against the runtime-d loop)
        for (uint32_t v = lane; v < nv; v += 32) {
            const uint2 lo = *reinterpret_cast<const uint2 *>(reinterpret_cast<const char *>(s4 + v) + 8);
            const uint2 hi = *reinterpret_cast<const uint2 *>(s4 + v + 1);
            st16(d4 + v, make_uint4(lo.x, lo.y, hi.x, hi.y));
        }
    } else {
        // the shift a compile-time constant in the loop (one loop per d)
        switch (d) {
#define MPXA_SHIFT_CASE(D) case D: shift_loop<D>(s4, d4, nv, lane); break;
            MPXA_SHIFT_CASE(1) MPXA_SHIFT_CASE(2) MPXA_SHIFT_CASE(3) MPXA_SHIFT_CASE(4)
            MPXA_SHIFT_CASE(5) MPXA_SHIFT_CASE(6) MPXA_SHIFT_CASE(7) MPXA_SHIFT_CASE(9)
            MPXA_SHIFT_CASE(10) MPXA_SHIFT_CASE(11) MPXA_SHIFT_CASE(12) MPXA_SHIFT_CASE(13)
            MPXA_SHIFT_CASE(14) default: shift_loop<15>(s4, d4, nv, lane); break;
#undef MPXA_SHIFT_CASE
        }
    }
    for (uint32_t i = hd + nv * 16 + lane; i < n; i += 32) dst[i] = stage[sh + i];
}

// Warp-ring dynamic mode, one tile: the tile's pieces (TMA queue first, then the rest) are
// taken from ONE work queue by the CTA's warps, each running its own pipeline: lane 0 keeps
// up to kWStages - 2 TMA bulk loads in flight (16-B aligned spans) into the warp's ring; the
// warp then drains the oldest stage -- a bulk store for a congruent piece, or 16-B stores
// shifted out of shared memory by the whole warp for a piece whose source and destination
// are not 16-B congruent (the LSU path's register-bound loads become TMA loads).  Pieces
// shorter than kTmaMin, and shifted fan-out pieces, go through lsu_copy.
__device__ __noinline__ bool dyn_tile_w(const ExecParams &P, ExecShared &S, int g, int first, int nm, bool loaded,
                                        bool classified, int ti) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t U = (uint64_t)P.dyn_u;
    if (!classified) dyn_classify(P, S, g, first, nm, loaded);
    CTA_STAMP(4);
    const uint32_t totA = S.pcA[nm], tot = totA + S.pcB[nm];
    if (tot == 0) return false;
    extern __shared__ __align__(128) char dyn_smem[];
    char *ring = dyn_smem + (size_t)w * kWStages * kWChunk;
    uint32_t *q = &P.dc->dyn_next[g * kMaxDynTiles + ti];
    bool wrote = false;
    const uint32_t base = S.wseq[w];   // ring position where this tile starts (all lanes)
    // lane 0's producer state; the next piece index is requested while the current streams
    uint32_t issued = 0, consumed = 0;
    bool have = false, exhausted = false;
    uint32_t nextu = lane == 0 ? atomicAdd(q, 1u) : 0u;
    int mi = 0;
    bool isA = false;
    MovePlan mp;
    uint64_t off = 0, end = 0;
    int lsu_mi = -1;             // a piece for lsu_copy by the whole warp (broadcast)
    uint64_t lsu_lo = 0;
    for (;;) {
        if (lane == 0) {
            // at most kWStages - P.wslack loads in flight: the stages behind them may still be
            // draining their bulk stores, so re-arming a stage rarely waits for one
            while (!exhausted && lsu_mi < 0 && issued - consumed < (uint32_t)(kWStages - P.wslack)) {
                if (!have) {
                    const uint32_t u = nextu;
                    if (u >= tot) { exhausted = true; break; }
                    nextu = atomicAdd(q, 1u);
                    isA = u < totA;
                    const uint32_t *pc = isA ? S.pcA : S.pcB;
                    const uint32_t uu = isA ? u : u - totA;
                    mi = find_move(pc, nm, uu);
                    const uint64_t lo = (uint64_t)(uu - pc[mi]) * U;
                    mp = piece_plan(P, S, mi, lo, U);
                    const Move &m = S.moves[mi];
                    if (!isA && (mp.n < kTmaMin || m.fanout)) {   // warp lsu_copy, outside the ring
                        lsu_mi = mi;
                        lsu_lo = lo;
                        break;
                    }
                    if (isA) {
                        uint64_t head = (16 - ((uintptr_t)mp.src & 15)) & 15;
                        if (head > mp.n) head = mp.n;
                        const uint64_t body = (mp.n - head) & ~(uint64_t)15;
                        if (head) { copy_edge(P, S, m, mp, 0, (uint32_t)head); wrote = true; }
                        if (mp.n > head + body) {
                            copy_edge(P, S, m, mp, head + body, (uint32_t)(mp.n - head - body));
                            wrote = true;
                        }
                        off = head;
                        end = head + body;
                    } else {
                        off = 0;
                        end = mp.n;
                    }
                    have = off < end;
                    if (!have) continue;
                }
                const uint32_t s = (base + issued) % (uint32_t)kWStages;
                ExecShared::WEntry &e = S.went[w][s];
                const Move &m = S.moves[mi];
                uint64_t len;
                const char *lsrc;
                if (isA) {
                    len = end - off < (uint64_t)kWChunk ? end - off : (uint64_t)kWChunk;
                    lsrc = mp.src + off;
                    e.kind = 0;
                    e.src = lsrc;
                    e.lbytes = (uint32_t)len;
                    e.sh = 0;
                    e.fanout = m.fanout;
                    e.dst_kind = m.dst_kind;
                    e.doff = mp.doff + off;
                    e.dst = m.fanout ? nullptr : mp.dst + off;
                } else {
                    // chunks end at 128-B (line) boundaries of the destination (except the
                    // piece's last), so no line is written half by one stage, half by the next
                    len = end - off < (uint64_t)(kWChunk - 32) ? end - off : (uint64_t)(kWChunk - 32);
                    if (off + len < end) len -= ((uintptr_t)(mp.dst + off + len)) & 127;
                    const uintptr_t s0 = (uintptr_t)(mp.src + off), a0 = s0 & ~(uintptr_t)15;
                    lsrc = (const char *)a0;
                    e.kind = 1;
                    e.src = mp.src + off;
                    e.lbytes = (uint32_t)(((s0 + len + 15) & ~(uintptr_t)15) - a0);
                    e.sh = (uint16_t)(s0 - a0);
                    e.fanout = 0;
                    e.dst_kind = m.dst_kind;
                    e.doff = 0;
                    e.dst = mp.dst + off;
                }
                e.n = (uint32_t)len;
                // the stage's previous contents: consumed, and its bulk store (if any) has
                // read shared memory -- one bulk group was committed per consumed entry
                if (issued >= (uint32_t)kWStages) bulk_wait_read((int)(consumed - 1 - (issued - kWStages)));
                tma_load_1d(smem_u32(ring + (size_t)s * kWChunk), lsrc, e.lbytes, smem_u32(&S.wmbar[w][s]));
                issued++;
                off += len;
                if (off >= end) have = false;
            }
        }
        issued = __shfl_sync(0xffffffffu, issued, 0);
        exhausted = __shfl_sync(0xffffffffu, exhausted, 0);
        lsu_mi = __shfl_sync(0xffffffffu, lsu_mi, 0);
        if (consumed == issued) {
            if (lsu_mi >= 0) {           // ring drained: the pending lsu_copy piece, whole warp
                lsu_lo = __shfl_sync(0xffffffffu, lsu_lo, 0);
                const MovePlan lp = piece_plan(P, S, lsu_mi, lsu_lo, U);
                lsu_copy(P, S, S.moves[lsu_mi], lp, 0, lp.n, lane, 32);
                wrote = true;
                lsu_mi = -1;
                __syncwarp();
                continue;
            }
            if (exhausted) break;
            continue;
        }
        __syncwarp();   // lane 0's stage descriptor before every lane reads it
        const uint32_t s = (base + consumed) % (uint32_t)kWStages;
        mbar_wait(smem_u32(&S.wmbar[w][s]), ((base + consumed) / (uint32_t)kWStages) & 1u);
#ifdef MPXA_TRACE
        if (consumed == 0 && w == 0) CTA_STAMP(5);
#endif
        const ExecShared::WEntry &e = S.went[w][s];
        const char *stage = ring + (size_t)s * kWChunk;
        if (e.kind == 0) {
            if (lane == 0) {
                if (!e.fanout) {
                    tma_store_1d(e.dst, smem_u32(stage), e.n);
                } else {
                    fan_store(P, S, e.dst_kind, e.doff, smem_u32(stage), e.n);
                }
            }
        } else {
            wring_shift_store(stage, e.sh, e.dst, e.n, lane);
            wrote = true;
        }
        __syncwarp();   // every lane's shared-memory reads of the stage are done
        if (lane == 0) bulk_commit();
        consumed++;
    }
    if (lane == 0) {
        bulk_wait_all();   // this warp's bulk stores complete (the step end fences)
        S.wseq[w] = base + issued;
    }
    __syncwarp();
    return wrote;
}

// Dynamic mode over the whole step: move tiles in order, each with its own pair of queues; a
// CTA moves on to the next tile as soon as the current tile's queues are dry (no barrier).
__device__ __noinline__ bool dyn_step(const ExecParams &P, ExecShared &S, Producer &prod, int g, int first, int nm,
                                      bool loaded, bool classified, int tile0) {
    bool wrote = false;
    for (int tile = 0, ti = tile0; tile < nm; tile += kMoveTile, ti++) {
        const int cnt = min(kMoveTile, nm - tile);
        const bool l0 = loaded && tile == 0, c0 = classified && tile == 0;
        wrote |= P.wring ? dyn_tile_w(P, S, g, first + tile, cnt, l0, c0, ti)
                         : dyn_tile(P, S, prod, g, first + tile, cnt, l0, c0, ti);
    }
    return wrote;
}

// Multi-step dynamic mode: every CTA of this GPU row has finished step s (its writes complete
// and fenced) -- a counter barrier; the grid never exceeds the co-resident CTA count.
__device__ __noinline__ void row_barrier(const ExecParams &P, ExecShared &S, int g, int s) {
    if (threadIdx.x == 0) {
        uint32_t *bar = &P.dc->dyn_bar[g];
        red_release_gpu_add(bar, 1u);
        const uint32_t want = (uint32_t)(s + 1) * gridDim.x;
        uint64_t t0 = 0;
        int it = 0;
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v >= want) break;
            if (++it > 16) {
                __nanosleep(64);
                if (!t0) t0 = globaltimer();
                else if ((int64_t)(globaltimer() - t0) > P.timeout_ns) { atomicExch(P.err, 1); S.abort_flag = 1; break; }
            }
        }
        fence_proxy_async();   // other CTAs' writes, acquired, before this CTA's TMA reads
    }
    __syncthreads();
}

#ifndef MPXA_EXEC_MINB
#define MPXA_EXEC_MINB 2
#endif
// DYN: dynamic (work-queue) mode, P.dyn_units != 0 -- its own instantiation, so the static
// mode's code stays compact
template <bool DYN>
__global__ void __launch_bounds__(kThreads, MPXA_EXEC_MINB) mpxa_exec_kernel(const __grid_constant__ ExecParams Pk) {
    extern __shared__ __align__(128) char dyn_smem[];
    __shared__ ExecShared S;
    // the helpers take the parameters by reference; a shared-memory copy keeps those
    // references out of the (slow, generic-addressed) kernel-parameter window
    __shared__ ExecParams P;
    CTA_STAMP(0);
    static_assert(sizeof(ExecParams) % 8 == 0, "ExecParams copy");
    for (int i = threadIdx.x; i < (int)(sizeof(ExecParams) / 8); i += kThreads)
        reinterpret_cast<uint64_t *>(&P)[i] = reinterpret_cast<const uint64_t *>(&Pk)[i];
    __syncthreads();
    TRACE(0);
    const int g = P.my_gpu >= 0 ? P.my_gpu : (int)blockIdx.y;
    const int c = blockIdx.x;
    const int sl = c % P.nS;                  // column slice
    const int f = c / P.nS;                   // flow group
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const GpuProg prog = P.mode == 1 ? P.progs[g] : P.prog;
    const bool multi = P.G > 1;   // emulated or multi-process: flags + CTS
    Producer prod;
    prod.stages = dyn_smem;

    const int64_t x0 = (int64_t)f * P.nflows / P.nF, x1 = (int64_t)(f + 1) * P.nflows / P.nF;
    const int nsteps = prog.nsteps;
    const bool steps_in_smem = nsteps <= kMaxStepsSmem;
    // Prologue: every bookkeeping load of the launch (step table, step 0's first move tile,
    // workspace / symmetric-region bases, epoch) is ISSUED before any is consumed -- one
    // memory round trip instead of a chain of them (these launches are latency-bound).
    const bool ld_step = steps_in_smem && t < nsteps;
    Step st_r;
    if (ld_step) st_r = prog.steps[t];
    // step 0 dense: its moves start at index 0 of every GPU's move array, so this CTA's
    // first move tile is known without the step table
    const bool pre = steps_in_smem && nsteps > 0 && P.d0_base >= 0;
    int pre_cnt = 0;
    Move mv_r;
    if (pre) {
        const int a = clampi(x0 - P.d0_base, P.d0_n);
        const int nm = clampi(x1 - P.d0_base, P.d0_n) - a;
        const int rot = (nm && !DYN) ? (int)(((int64_t)sl + (int64_t)g * nm / P.G) % nm) : 0;
        pre_cnt = min(kMoveTile, nm);            // <= kThreads: one move per thread
        if (t < pre_cnt) {
            int q = t + rot;
            if (q >= nm) q -= nm;
            mv_r = prog.moves[a + q];
        }
    }
    char *wb_r = nullptr;
    SymRegion *sym_r = nullptr;
    if (t < P.G) {
        wb_r = P.dc->work_base[t];
        sym_r = P.dc->sym[t];
    }
    if (t == kThreads - 1) {    // a thread with no load outstanding (the fence is a release)
        if (P.wring) {
            for (int w = 0; w < kWarpsExec; w++)
                for (int s = 0; s < kWStages; s++) mbar_init(smem_u32(&S.wmbar[w][s]), 1);
        } else {
            for (int s = 0; s < P.stages; s++) mbar_init(smem_u32(&S.mbar[s]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    TRACE(9);
    if (ld_step) {
        if (P.nF == 1) {            // one flow group: the whole step, no flow-index lookup
            S.steps[t] = StepInfo{st_r.move_begin, st_r.move_end - st_r.move_begin, st_r.signal_mask, st_r.wait_mask};
        } else if (P.dyn_sync) {    // steps end at a row barrier: no cross-step ownership, so the
                                    // GPU's own moves split evenly (global flow ranges would leave
                                    // all but 1/G of the flow groups idle on each GPU)
            const int n = st_r.move_end - st_r.move_begin;
            const int a = (int)((int64_t)n * f / P.nF), b = (int)((int64_t)n * (f + 1) / P.nF);
            S.steps[t] = StepInfo{st_r.move_begin + a, b - a, st_r.signal_mask, st_r.wait_mask};
        } else if (st_r.dense_base >= 0) {   // move k carries flow dense_base + k: arithmetic range
            const int n = st_r.move_end - st_r.move_begin;
            const int a = clampi(x0 - st_r.dense_base, n);
            const int b = clampi(x1 - st_r.dense_base, n);
            S.steps[t] = StepInfo{st_r.move_begin + a, b - a, st_r.signal_mask, st_r.wait_mask};
        } else {
            const int32_t *fx = prog.findex + st_r.flow_index;
            const int m0 = fx[x0];
            S.steps[t] = StepInfo{st_r.move_begin + m0, fx[x1] - m0, st_r.signal_mask, st_r.wait_mask};
        }
    }
    if (t < pre_cnt) S.moves[t] = mv_r;
    if (t < P.G) {
        S.work_base[t] = wb_r;
        S.sym[t] = sym_r;
        // own / local recv bases; remote ones (emulated, multi-process) arrive with the CTS
        S.recv_base[t] = P.mode == 0 ? P.recv
                         : P.mode == 1 ? (t == g ? P.recv + (uint64_t)t * P.R * P.recv_stride : nullptr)
                                       : (t == g ? P.recv : nullptr);
    }
    if (t == 0) {
        S.cts_ok = 0;
        S.abort_flag = 0;
    }
    if (t < kWarpsExec) S.wseq[t] = 0;
    TRACE(10);
    __syncthreads();
    // Dynamic mode on one GPU: step 0's first move tile (prefetched above) is classified and
    // its piece prefixes scanned BEFORE the dependency wait -- it reads only this launch's
    // moves, parameters and buffer bases, nothing a previous kernel writes -- so the ~2 us
    // of cold-instruction classification overlaps the previous kernel's tail (measured, p = 8
    // allgather 4 MiB: wait -> first piece 2.4 us, MPXA_TRACE build, tools/ag_trace2.py).
    // Peers' bases (several GPUs) arrive with the CTS after the wait: classified there.  A
    // step 0 that is not dense (alltoallv) has its first tile loaded here first (program
    // tables are this launch's: persistent, or uploaded before a launch without PDL).
    const bool pre_cls = DYN && steps_in_smem && !multi && nsteps > 0;
    if (pre_cls) {
        const int nm0 = min(kMoveTile, S.steps[0].nm);
        if (!pre) {
            if (t < nm0) S.moves[t] = prog.moves[S.steps[0].first + t];
            __syncthreads();
        }
        const uint32_t k0 = dyn_classify(P, S, g, S.steps[0].first, nm0, true);
        if (t == 0) S.kuni0 = k0;
    }
    griddep_wait();
    griddep_launch_dependents();
    CTA_STAMP(2);
    if (multi) {
        if (t == 0) S.epoch = *(volatile uint64_t *)&P.dc->epoch + 1;
        __syncthreads();
    }
    TRACE(14);
    const uint64_t epoch = S.epoch;
    // CTS: this GPU is inside `epoch`, so every earlier use of its buffers is complete
    // (stream order); tell every peer it may write into them, and where its recvbuf is
    // (registered window + offset; emulated GPUs: window 0 has base 0, offset = address).
    if (multi && c == 0 && t < P.G && t != g) {
        CtsSlot *slot = &S.sym[t]->cts[g];
        if (P.mode == 2) { slot->win = P.recv_win; slot->off = P.recv_off; }
        else { slot->win = 0; slot->off = (uint64_t)(uintptr_t)(P.recv + (uint64_t)g * P.R * P.recv_stride); }
        st_release_sys(&slot->epoch, epoch);
    }

    SliceCache sc;
    int tile_base = 0;   // dynamic mode: first queue tile of the current step
    TRACE(1);
    for (int s = 0; s < nsteps; s++) {
        StepInfo st;
        if (steps_in_smem) {
            st = S.steps[s];
        } else {
            const Step g_st = prog.steps[s];
            if (P.dyn_sync) {
                const int n = g_st.move_end - g_st.move_begin;
                const int a = (int)((int64_t)n * f / P.nF), b = (int)((int64_t)n * (f + 1) / P.nF);
                st = StepInfo{g_st.move_begin + a, b - a, g_st.signal_mask, g_st.wait_mask};
            } else {
                const int32_t *fx = prog.findex + g_st.flow_index;
                const int m0 = fx[x0];
                st = StepInfo{g_st.move_begin + m0, fx[x1] - m0, g_st.signal_mask, g_st.wait_mask};
            }
        }
        const uint32_t prev_wait = s == 0 ? 0u : (steps_in_smem ? S.steps[s - 1].wait_mask : prog.steps[s - 1].wait_mask);
        bool wrote = false;   // this thread issued generic global stores in this step
        const int fslot = P.dyn_sync ? 0 : c;   // flag slot: this CTA's, or the row's (sync mode)
        if (multi) {
            // data written into this GPU by peers in step s-1 (this CTA's share) must have landed
            if (prev_wait)
                wait_mask_ge(P, S, prev_wait, &S.sym[g]->flags[0][fslot], kMaxCtas, (epoch << 8) | (uint64_t)s);
            // peers written in this step must have cleared us to send in this epoch
            uint32_t need = st.signal_mask & ~S.cts_ok;
            if (need) {
                wait_mask_ge(P, S, need, &S.sym[g]->cts[0].epoch, sizeof(CtsSlot) / 8, epoch);
                if (t < 32 && ((need >> t) & 1u)) {
                    const CtsSlot *cs = &S.sym[g]->cts[t];
                    S.recv_base[t] = P.dc->win_table[t * kMaxWindows + cs->win] + cs->off;
                }
            }
            __syncthreads();
            if (t == 0) S.cts_ok |= need;
            if (S.abort_flag) return;
        }
        if (multi && t == 0) fence_proxy_async();   // acquired peer writes before TMA reads
        const int nm = DYN ? 0 : st.nm;   // dynamic mode: the work queue below
        const int rot = nm ? (int)(((int64_t)sl + (int64_t)g * nm / P.G) % nm) : 0;
        if (DYN) {
            wrote = dyn_step(P, S, prod, g, st.first, st.nm, (pre || pre_cls) && s == 0, pre_cls && s == 0, tile_base);
            tile_base += (st.nm + kMoveTile - 1) / kMoveTile;
        }
        for (int tile = 0; tile < nm; tile += kMoveTile) {
            const int cnt = min(kMoveTile, nm - tile);
            if (!(pre && s == 0 && tile == 0)) {   // (prefetched in the prologue)
                __syncthreads();   // the previous tile's moves are no longer read
                for (int i = t; i < cnt; i += kThreads) {
                    int q = tile + i + rot;
                    if (q >= nm) q -= nm;
                    S.moves[i] = prog.moves[st.first + q];
                }
                __syncthreads();
            }
            TRACE(2);
            if (warp == 0) {
                if (lane == 0) {
                    for (int i = 0; i < cnt; i++) {
                        const Move &m = S.moves[i];
                        uint64_t lo;
                        if (slice_len(P, m, sl, sc, lo) < kTmaMin) continue;   // cheap reject
                        const MovePlan mp = plan_move(P, S, m, sl, sc);
                        if (!mp.tma) continue;
                        const uint64_t chunk = (uint64_t)P.chunk;
                        for (uint64_t o = 0; o < mp.body; o += chunk) {
                            RingEntry e;
                            e.len = (uint32_t)min(chunk, mp.body - o);
                            e.fanout = m.fanout;
                            e.dst_kind = m.dst_kind;
                            e.doff = mp.doff + mp.head + o;
                            e.dst = m.fanout ? nullptr : mp.dst + mp.head + o;
                            prod.push(P, S, mp.src + mp.head + o, e);
                        }
                    }
                }
            } else {
                const int lw = warp - 1, lt = t - 32;
                SmallJob jobs[kBatch];
                int nj = 0;
                for (int i = 0; i < cnt; i++) {
                    const Move &m = S.moves[i];
                    uint64_t lo;
                    const uint64_t n = slice_len(P, m, sl, sc, lo);
                    // only the owning warp plans small moves; big ones involve every LSU thread
                    if (n == 0 || (n < kLsuBig && i % kLsuWarps != lw)) continue;
                    const MovePlan mp = plan_move(P, S, m, sl, sc);
                    if (mp.tma) {
                        if (i % kLsuWarps == lw) {   // head / tail bytes around the TMA body
                            const uint64_t tail = mp.n - mp.head - mp.body;
                            if (lane < 16) lsu_copy(P, S, m, mp, 0, mp.head, lane, 16);
                            else lsu_copy(P, S, m, mp, mp.head + mp.body, tail, lane - 16, 16);
                            wrote = true;
                        }
                    } else if (mp.n >= kLsuBig) {
                        lsu_copy(P, S, m, mp, 0, mp.n, lt, kLsuThreads);
                        wrote = true;
                    } else if (i % kLsuWarps == lw) {
                        if (mp.n <= kSmallMax) {     // batch small moves: one round trip per batch
                            jobs[nj].src = mp.src;
                            jobs[nj].dst = mp.dst;
                            jobs[nj].doff = mp.doff;
                            jobs[nj].n = (uint32_t)mp.n;
                            jobs[nj].fanout = m.fanout;
                            jobs[nj].dst_kind = m.dst_kind;
                            jobs[nj].ro = m.src_kind == BK_SEND;
                            if (++nj == kBatch) { small_batch(P, S, jobs, nj, lane); nj = 0; }
                        } else {
                            lsu_copy(P, S, m, mp, 0, mp.n, lane, 32);
                        }
                        wrote = true;
                    }
                }
                if (nj) small_batch(P, S, jobs, nj, lane);
            }
            TRACE(3);
        }
        // writers make their generic stores visible to the async proxy when anything will
        // consume them (a later step of this launch, or a peer signalled now); the producer
        // waits its bulk stores and fences them for generic readers
        const bool consumed = (s + 1 < nsteps) || (multi && st.signal_mask);
        if (consumed && wrote) fence_proxy_async();
        if (t == 0) prod.drain(P, S, consumed);
        TRACE(4);
        __syncthreads();
        TRACE(5);
        if (P.dyn_sync) {
            // every CTA of the row done with step s; then one signal per peer GPU
            if (s + 1 < nsteps || (multi && st.signal_mask)) row_barrier(P, S, g, s);
            if (S.abort_flag) return;
            if (multi && c == 0 && st.signal_mask && t < 32 && ((st.signal_mask >> t) & 1u)) {
                st_release_sys(&S.sym[t]->flags[g][0], (epoch << 8) | (uint64_t)(s + 1));
            }
            continue;
        }
        // ---- signal the peers written in this step (this CTA's share) ----
        if (multi && st.signal_mask && t < 32 && ((st.signal_mask >> t) & 1u)) {
            st_release_sys(&S.sym[t]->flags[g][c], (epoch << 8) | (uint64_t)(s + 1));
        }
    }
    // completion: everything peers write into this GPU in the last step has landed
    const uint32_t last_wait = nsteps == 0 ? 0u : (steps_in_smem ? S.steps[nsteps - 1].wait_mask
                                                                  : prog.steps[nsteps - 1].wait_mask);
    // (per-GPU signals: the peers' last-step data is complete when their one flag is; one
    // CTA waiting keeps the grid alive until then, the others retire and free their SMs)
    if (multi && last_wait && (!P.dyn_sync || c == 0)) {
        wait_mask_ge(P, S, last_wait, &S.sym[g]->flags[0][P.dyn_sync ? 0 : c], kMaxCtas,
                     (epoch << 8) | (uint64_t)nsteps);
        __syncthreads();
    }
    // the last CTA of the launch publishes the epoch and resets the work queues (the next
    // launch is stream-ordered after, and waits on griddepcontrol before reading either)
    if ((multi || DYN) && t == 0) {
        const uint32_t total = gridDim.x * gridDim.y;
        if (atom_acq_rel_gpu_add(&P.dc->done_ctas, 1u) == total - 1) {
            P.dc->done_ctas = 0;
            if (multi) P.dc->epoch = epoch;
            if (DYN || P.dyn_sync)
                for (int r = 0; r < (int)gridDim.y; r++) {
                    const int row = P.my_gpu >= 0 ? P.my_gpu : r;
                    for (int ti = 0; DYN && ti < P.dyn_units; ti++) {
                        P.dc->dyn_next[row * kMaxDynTiles + ti] = 0;
                        P.dc->dyn_next2[row * kMaxDynTiles + ti] = 0;
                    }
                    P.dc->dyn_bar[row] = 0;   // row barriers (dynamic or per-GPU-signalled steps)
                }
            // (no fence: the next launch reads these after griddepcontrol.wait / grid completion)
        }
    }
    CTA_STAMP(1);
}

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
// host-side launchers (called from api.cpp)
// ------------------------------------------------------------------------------------
// ------------------------------------------------------------------------------------
// Small-message executor (short moves): items are (move, 16-byte piece) pairs spread over
// all threads, four in flight per thread, moves cached in shared memory, no TMA and little
// code -- these launches are latency-bound, so the kernel touches as few instruction lines
// and memory round trips as possible.  Multi-step programs run in ONE CTA per GPU (steps
// are separated by __syncthreads); single-step programs may use several CTAs (no step
// reads another CTA's output).  Same program format and flag/CTS protocol as
// mpxa_exec_kernel (CTA c signals / waits slot c).
// ------------------------------------------------------------------------------------
constexpr int kSmallThreads = 512;


struct SmallShared {
    StepInfo steps[kMaxStepsSmem];   // step table, loaded in the prologue (before griddep wait)
    uint32_t n_own;                  // owned-flow mode: moves of this step owned by this CTA
    char *rb[3][kRankTable];         // [kind][rank] buffer base (p <= kRankTable): no divisions
    char *recv_base[kMaxGpus];
    char *work_base[kMaxGpus];
    SymRegion *sym[kMaxGpus];
    uint64_t epoch;
    uint32_t cts_ok;
    int abort_flag;
    uint64_t ll_seq;                 // eager mode: this launch's sequence number (the flag) ...
    uint64_t ll_par;                 // ... and the byte offset of its staging parity
};

__device__ __forceinline__ char *sbase(const ExecParams &P, const SmallShared &S, int kind, int rank) {
    const int g = rank / P.R;
    const uint64_t local = (uint64_t)(rank - g * P.R);
    if (kind == BK_SEND)
        return (char *)P.send + (P.mode == 2 ? 0 : (uint64_t)g * P.R * P.send_stride) + local * P.send_stride;
    if (kind == BK_RECV) return S.recv_base[g] + local * P.recv_stride;
    return S.work_base[g] + local * P.work_stride;
}

__device__ __forceinline__ char *sb(const ExecParams &P, const SmallShared &S, int kind, int rank) {
    return P.p <= kRankTable ? S.rb[kind][rank] : sbase(P, S, kind, rank);
}
// (re)fill the rank-base rows of the ranks on GPUs in gmask (threads t < p)
__device__ __forceinline__ void fill_rank_bases(const ExecParams &P, SmallShared &S, uint32_t gmask, bool all_kinds) {
    const int t = threadIdx.x;
    if (P.p > kRankTable || t >= P.p) return;
    const int gg = t / P.R;
    if (!((gmask >> gg) & 1u)) return;
    if (all_kinds) {
        S.rb[BK_SEND][t] = sbase(P, S, BK_SEND, t);
        S.rb[BK_WORK][t] = sbase(P, S, BK_WORK, t);
    }
    S.rb[BK_RECV][t] = S.recv_base[gg] ? sbase(P, S, BK_RECV, t) : nullptr;
}

// threads < 32, one per set bit of mask: spin until slot >= want (watchdog as in the main kernel)
__device__ __forceinline__ void small_wait(const ExecParams &P, SmallShared &S, uint32_t mask, const uint64_t *slot0,
                                           uint64_t stride, uint64_t want) {
    const int t = threadIdx.x;
    if (t < 32 && ((mask >> t) & 1u)) {
        const uint64_t *slot = slot0 + (uint64_t)t * stride;
        uint64_t start = 0;
        int it = 0;
        while (ld_acquire_sys(slot) < want) {
            if (++it > 32) {
                __nanosleep(64);
                if (start == 0) start = globaltimer();
                else if ((int64_t)(globaltimer() - start) > P.timeout_ns) {
                    atomicExch(P.err, 1);
                    S.abort_flag = 1;
                    break;
                }
            }
            if (*(volatile int *)&S.abort_flag) break;
        }
    }
}

// multi-step small launches over several CTAs (ExecParams::dyn_sync): the CTAs of a GPU row
// meet at a counter barrier between steps (every CTA of the launch is co-resident)
__device__ __noinline__ void small_row_barrier(const ExecParams &P, SmallShared &S, int g, int s) {
    if (threadIdx.x == 0) {
        uint32_t *bar = &P.dc->dyn_bar[g];
        red_release_gpu_add(bar, 1u);
        const uint32_t want = (uint32_t)(s + 1) * gridDim.x;
        uint64_t t0 = 0;
        int it = 0;
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v >= want) break;
            if (++it > 16) {
                __nanosleep(32);
                if (!t0) t0 = globaltimer();
                else if ((int64_t)(globaltimer() - t0) > P.timeout_ns) { atomicExch(P.err, 1); S.abort_flag = 1; break; }
            }
        }
    }
    __syncthreads();
}

// items = (move, 16-byte piece); thread takes items base0, base0 + TT, ... kBatch at a time
// VAR: items are the exact pieces of a warp's tile of 32 moves mv[] (exclusive piece prefix
// vpc[]): the move is the last j with vpc[j] <= it (moves past the tile's end carry the
// tile total, zero-length ones share their successor's prefix and lose the search)
template <bool VAR>
__device__ __forceinline__ const Move &item_move(const Move *mv, const uint16_t *idx, const uint32_t *vpc, uint32_t it,
                                                 uint32_t lg, uint32_t mask, uint32_t &o) {
    if (VAR) {
        int j = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1)   // j + step <= 31 throughout
            if (vpc[j + step] <= it) j += step;
        o = (it - vpc[j]) * 16;
        return mv[j];
    }
    o = (it & mask) * 16;
    return mv[idx ? idx[it >> lg] : (it >> lg)];
}

template <int AW, bool VAR = false>
__device__ __forceinline__ void small_items(const ExecParams &P, const SmallShared &S, const Move *mv, uint32_t items,
                                            uint32_t lg, uint32_t TT, uint32_t base0, const uint16_t *idx,
                                            const uint32_t *vpc = nullptr) {
    const uint32_t mask = (1u << lg) - 1u;   // pieces per move: a power of two (host-rounded)
    for (uint32_t base = base0; base < items; base += TT * kBatch) {
        PieceRegs<AW> R;
        const char *sp[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; k++) {
            sp[k] = nullptr;
            const uint32_t it = base + (uint32_t)k * TT;
            if (it >= items) continue;
            uint32_t o;
            const Move &m = item_move<VAR>(mv, idx, vpc, it, lg, mask, o);
            if (k == 0) TRACE(13);
            const uint32_t n = (uint32_t)((uint64_t)m.len * P.unit);
            if (o >= n) continue;
            sp[k] = sb(P, S, m.src_kind, m.src_rank) + (uint64_t)m.src_off * P.unit + o;
            R.issue(k, sp[k], min(16u, n - o));
        }
        TRACE(1);
#pragma unroll
        for (int k = 0; k < kBatch; k++) {
            if (!sp[k]) continue;
            const uint32_t it = base + (uint32_t)k * TT;
            uint32_t o;
            const Move &m = item_move<VAR>(mv, idx, vpc, it, lg, mask, o);
            const uint32_t n = (uint32_t)((uint64_t)m.len * P.unit);
            const uint32_t len = min(16u, n - o);
            const uint64_t doff = (uint64_t)m.dst_off * P.unit + o;
            const uint4 val = R.value(k, sp[k]);
            if (!m.fanout) {
                store_piece<AW>(sb(P, S, m.dst_kind, m.dst_rank) + doff, val, len);
            } else {
#pragma unroll 1
                for (int r = 0; r < P.p; r++) store_piece<AW>(sb(P, S, m.dst_kind, r) + doff, val, len);
            }
        }
    }
}

// kSmallLocal with P.small_swork: the WORK rows after the cached moves (16-B aligned)
__host__ __device__ __forceinline__ size_t swork_offset(const ExecParams &P) {
    return ((size_t)P.small_cache * sizeof(Move) + 15) / 16 * 16;
}

// Single-GPU launches with every move cached (kSmallLocal): each move is resolved ONCE, in the
// prologue, to absolute source / destination pointers and a byte count, in place of the cached
// Move -- the per-item path is then one shared-memory record and no base-table lookups.
struct RMove {
    const char *src;
    char *dst;         // non-fanout destination
    uint64_t doff;     // fanout: byte offset inside every rank's dst_kind buffer
    uint32_t n;        // bytes
    uint32_t flow;
    uint8_t fanout, dst_kind;
    uint8_t src_sm, dst_sm;   // source / destination in shared memory (P.small_swork)
    uint8_t dst_remote;       // destination on a peer GPU: base from the CTS-filled table at store
    uint8_t ll;               // eager mode: 1 = send words to dst (peer staging, parity 0 address),
                              // 2 = receive words from src (own staging); fanout 2 = own ranks only
    uint16_t dst_rank;
};
static_assert(sizeof(RMove) == sizeof(Move), "resolved moves overwrite the cached moves 1:1");

// buffer base of `rank`, a rank of this CTA's GPU g (every move reads there; destinations on
// g too), from the launch parameters alone
__device__ __forceinline__ char *local_base(const ExecParams &P, int g, char *work_g, int kind, int rank) {
    const uint64_t local = (uint64_t)(rank - g * P.R);
    if (kind == BK_SEND)
        return (char *)P.send + (P.mode == 2 ? 0 : (uint64_t)g * P.R * P.send_stride) + local * P.send_stride;
    if (kind == BK_RECV) return P.recv + (P.mode == 1 ? (uint64_t)g * P.R * P.recv_stride : 0) + local * P.recv_stride;
    return work_g + local * P.work_stride;
}

template <int AW>
__device__ __forceinline__ void small_items_loc(const ExecParams &P, const SmallShared &S, const RMove *mv,
                                                uint32_t items, uint32_t lg, uint32_t TT, uint32_t base0,
                                                const uint16_t *idx) {
    const uint32_t mask = (1u << lg) - 1u;
    for (uint32_t base = base0; base < items; base += TT * kBatch) {
        PieceRegs<AW> R;
        const char *sp[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; k++) {
            sp[k] = nullptr;
            const uint32_t it = base + (uint32_t)k * TT;
            if (it >= items) continue;
            const RMove &m = mv[idx ? idx[it >> lg] : (it >> lg)];
            const uint32_t o = (it & mask) * 16;
            if (o >= m.n) continue;
            sp[k] = m.src + o;
            if (m.src_sm) R.issue_generic(k, sp[k], min(16u, m.n - o));
            else R.issue(k, sp[k], min(16u, m.n - o));
        }
        TRACE(1);
#pragma unroll
        for (int k = 0; k < kBatch; k++) {
            if (!sp[k]) continue;
            const uint32_t it = base + (uint32_t)k * TT;
            const RMove &m = mv[idx ? idx[it >> lg] : (it >> lg)];
            const uint32_t o = (it & mask) * 16;
            const uint32_t len = min(16u, m.n - o);
            const uint4 val = R.value(k, sp[k]);
            if (m.dst_sm) {
                store_piece_generic(m.dst + o, val, len);
            } else if (!m.fanout) {
                store_piece<AW>((m.dst_remote ? S.rb[m.dst_kind][m.dst_rank] + m.doff : m.dst) + o, val, len);
            } else {
#pragma unroll 1
                for (int r = 0; r < P.p; r++) store_piece_generic(S.rb[m.dst_kind][r] + m.doff + o, val, len);
            }
        }
    }
}

__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// two eager words {data0, flag, data1, flag} in one 16-byte store; each 8-byte half is written
// atomically, so the receiver checks both flags (the 16 bytes as a whole are not atomic)
__device__ __forceinline__ void st_ll_pair(uint64_t *p, uint32_t d0, uint32_t d1, uint32_t flag) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(d0), "r"(flag), "r"(d1), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_ll_pair(const uint64_t *p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}

// Eager (LL) mode, one phase of a step (P.small_ll).  RECV = false: local moves
// and sends -- a send piece stores its (up to) four payload words, each with the launch's flag
// in the high half, into the peer's staging (no fence: every 8-byte word is its own signal).
// RECV = true: receive pieces poll their words in this GPU's staging until all carry the flag,
// then store the payload to the destination (fan-out 2: every rank of this GPU).  Flag-only
// moves (n = 0) send / await one word.
template <bool A16, bool RECV>
__device__ __forceinline__ void small_items_ll(const ExecParams &P, SmallShared &S, const RMove *mv, uint32_t items,
                                               uint32_t lg, uint32_t TT, uint32_t base0, int g) {
    const uint32_t mask = (1u << lg) - 1u;
    const uint64_t flag = S.ll_seq << 32, par = S.ll_par;
    for (uint32_t base = base0; base < items; base += TT * kBatch) {
        PieceRegs<A16 ? 16 : 0> R;
        uint4 lv[kBatch];
        bool on[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; k++) {
            on[k] = false;
            const uint32_t it = base + (uint32_t)k * TT;
            if (it >= items) continue;
            const RMove &m = mv[it >> lg];
            const uint32_t o = (it & mask) * 16;
            if (o >= m.n && !(m.ll && o == 0)) continue;
            on[k] = true;
            if (RECV) continue;
            if (o < m.n) R.issue(k, m.src + o, min(16u, m.n - o));
        }
        if (RECV) {   // poll: all words of the piece carry this launch's flag
#pragma unroll
            for (int k = 0; k < kBatch; k++) {
                if (!on[k]) continue;
                const uint32_t it = base + (uint32_t)k * TT;
                const RMove &m = mv[it >> lg];
                const uint32_t o = (it & mask) * 16;
                const uint32_t nw = m.n > o ? (min(16u, m.n - o) + 3) / 4 : 1;
                const uint64_t *w = reinterpret_cast<const uint64_t *>(m.src + par) + o / 4;   // 16-B aligned
                const uint32_t f32 = (uint32_t)(flag >> 32);
                uint32_t d[4] = {0, 0, 0, 0};
                uint64_t t0 = 0;
                for (uint32_t j = 0; j < nw; j += 2) {   // word pairs: one 16-byte load each
                    uint4 v = ld_ll_pair(w + j);
                    int spins = 0;
                    while (v.y != f32 || (j + 1 < nw && v.w != f32)) {
                        if (++spins > 64) {
                            __nanosleep(64);
                            if (!t0) t0 = globaltimer();
                            else if ((int64_t)(globaltimer() - t0) > P.timeout_ns) {
                                atomicExch(P.err, 1);
                                S.abort_flag = 1;
                                return;
                            }
                        }
                        v = ld_ll_pair(w + j);
                    }
                    d[j] = v.x;
                    if (j + 1 < 4) d[j + 1] = v.z;
                }
                lv[k] = make_uint4(d[0], d[1], d[2], d[3]);
            }
        }
#pragma unroll
        for (int k = 0; k < kBatch; k++) {
            if (!on[k]) continue;
            const uint32_t it = base + (uint32_t)k * TT;
            const RMove &m = mv[it >> lg];
            const uint32_t o = (it & mask) * 16;
            const uint32_t len = m.n > o ? min(16u, m.n - o) : 0u;
            if (!RECV && m.ll == 1) {   // send: payload words + flag into the peer's staging
                const uint4 val = len ? R.value(k, m.src + o) : make_uint4(0, 0, 0, 0);
                uint64_t *w = reinterpret_cast<uint64_t *>(m.dst + par) + o / 4;   // 16-B aligned
                const uint32_t d[4] = {val.x, val.y, val.z, val.w};
                const uint32_t nw = len ? (len + 3) / 4 : 1, f32 = (uint32_t)(flag >> 32);
                for (uint32_t j = 0; j < nw; j += 2) {
                    if (j + 1 < nw) st_ll_pair(w + j, d[j], d[j + 1], f32);
                    else st_relaxed_sys(w + j, flag | d[j]);
                }
                continue;
            }
            if (!len) continue;
            const uint4 val = RECV ? lv[k] : R.value(k, m.src + o);
            if (m.fanout == 2) {
#pragma unroll 1
                for (int r = g * P.R; r < (g + 1) * P.R; r++) store_piece<A16 ? 16 : 0>(S.rb[m.dst_kind][r] + m.doff + o, val, len);
            } else {
                store_piece<A16 ? 16 : 0>(m.dst + o, val, len);
            }
        }
    }
}

// Variable-piece mode (P.small_var): one step of the small kernel.
__device__ __forceinline__ void small_var_step(const ExecParams &P, const SmallShared &S, const Move *mvs, int first,
                                            int nm, bool a16, char *small_dyn) {
    const int t = threadIdx.x;
    // warp tiles of 32 moves, round-robin over the grid's warps: one move per lane, a
    // shuffle scan of their piece counts, then the lanes share the tile's pieces (no
    // block barrier; the host split long moves so tiles carry comparable work).  The tile
    // and its exclusive piece prefix live in dynamic shared memory after the cached moves.
    const int lane = t & 31, warp = t >> 5;
    Move *wm = reinterpret_cast<Move *>(small_dyn + (size_t)P.small_cache * sizeof(Move)) + warp * 32;
    uint32_t *wp = reinterpret_cast<uint32_t *>(small_dyn + (size_t)(P.small_cache + kSmallThreads) * sizeof(Move)) +
                   warp * 32;
    const int nwt = (nm + 31) >> 5, W = kSmallThreads / 32;
    for (int wt = (int)blockIdx.x * W + warp; wt < nwt; wt += (int)gridDim.x * W) {
        __syncwarp();   // the previous tile is no longer read
        const int i = wt * 32 + lane;
        uint32_t pcs = 0;
        if (i < nm) {
            const Move m = mvs[first + i];
            wm[lane] = m;
            pcs = (uint32_t)(((uint64_t)m.len * P.unit + 15) / 16);
        }
        uint32_t inc = pcs;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o2);
            if (lane >= o2) inc += y;
        }
        wp[lane] = inc - pcs;
        const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
        __syncwarp();
        if (a16) small_items<16, true>(P, S, wm, tot, 0, 32, lane, nullptr, wp);
        else small_items<0, true>(P, S, wm, tot, 0, 32, lane, nullptr, wp);
    }
}

// VARK: the variable-piece instantiation (P.small_var), a kernel of its own -- compiled into
// the common one its code cost every small launch ~8 % (registers / code layout, measured)
// Cold per-step paths of the small kernel, kept out of line so the single-GPU step loop stays
// compact in the instruction cache (measured: small launches are bound by per-step latency,
// not by bytes).  Every thread of the CTA calls them.
//
// Step entry across GPUs: the peers' flags for the previous step and the CTS of the GPUs this
// step writes to (their recv bases arrive with it).  Returns false after a watchdog abort.
__device__ __noinline__ bool small_step_enter(const ExecParams &P, SmallShared &S, int g, int s, uint32_t prev_wait,
                                              uint32_t signal_mask, uint64_t epoch, int fslot) {
    const int t = threadIdx.x;
    if (prev_wait) small_wait(P, S, prev_wait, &S.sym[g]->flags[0][fslot], kMaxCtas, (epoch << 8) | (uint64_t)s);
    const uint32_t need = signal_mask & ~S.cts_ok;
    if (need) {
        small_wait(P, S, need, &S.sym[g]->cts[0].epoch, sizeof(CtsSlot) / 8, epoch);
        if (t < 32 && ((need >> t) & 1u)) {
            const CtsSlot *cs = &S.sym[g]->cts[t];
            S.recv_base[t] = P.dc->win_table[t * kMaxWindows + cs->win] + cs->off;
        }
        __syncthreads();
        fill_rank_bases(P, S, need, false);
    }
    __syncthreads();
    if (t == 0) S.cts_ok |= need;
    return !S.abort_flag;
}

// Kernel start across GPUs: post this GPU's clear-to-send (epoch, and the recv window) into
// every peer's symmetric region.
__device__ __noinline__ void small_post_cts(const ExecParams &P, SmallShared &S, int g, uint64_t epoch) {
    const int t = threadIdx.x;
    if (t < P.G && t != g) {
        CtsSlot *slot = &S.sym[t]->cts[g];
        if (P.mode == 2) { slot->win = P.recv_win; slot->off = P.recv_off; }
        else { slot->win = 0; slot->off = (uint64_t)(uintptr_t)(P.recv + (uint64_t)g * P.R * P.recv_stride); }
        st_release_sys(&slot->epoch, epoch);
    }
}

// Kernel end: the peers' flags of the last step, then the last CTA of the launch publishes the
// epoch and resets the sync-mode barrier counters (graph-replayable launches).
__device__ __noinline__ void small_finish(const ExecParams &P, SmallShared &S, int g, int nsteps, uint32_t prev_wait,
                                          uint64_t epoch) {
    const bool multi = P.G > 1;
    if (multi && prev_wait) {
        small_wait(P, S, prev_wait, &S.sym[g]->flags[0][P.dyn_sync ? 0 : (int)blockIdx.x], kMaxCtas,
                   (epoch << 8) | (uint64_t)nsteps);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (atom_acq_rel_gpu_add(&P.dc->done_ctas, 1u) == gridDim.x * gridDim.y - 1) {
            P.dc->done_ctas = 0;
            if (multi) P.dc->epoch = epoch;
            if (P.small_ll) P.dc->ll_seq = S.ll_seq;
            if (P.dyn_sync)
                for (int r = 0; r < (int)gridDim.y; r++) P.dc->dyn_bar[P.mode == 1 ? r : P.my_gpu] = 0;
        }
    }
}

// Owned-flow mode: compact the indexes of this CTA's moves of the step into own[]; returns
// their number.
__device__ __noinline__ uint32_t small_own_list(const ExecParams &P, SmallShared &S, const Move *mv, int nm,
                                                uint16_t *own, bool resolved) {
    const int t = threadIdx.x;
    if (t == 0) S.n_own = 0;
    __syncthreads();
    for (int i = t; i < nm; i += (int)blockDim.x) {
        const uint32_t flow = resolved ? reinterpret_cast<const RMove *>(mv)[i].flow : mv[i].flow;
        if ((int)(flow % (uint32_t)P.small_own) == (int)blockIdx.x) own[atomicAdd(&S.n_own, 1u)] = (uint16_t)i;
    }
    __syncthreads();
    return S.n_own;
}

// Step exit: the row barrier of sync mode, then the step's flags to the GPUs it wrote.
// Returns false after a watchdog abort.
__device__ __noinline__ bool small_step_exit(const ExecParams &P, SmallShared &S, int g, int s, int nsteps,
                                             uint32_t signal_mask, uint64_t epoch, int fslot) {
    const int t = threadIdx.x;
    const bool multi = P.G > 1;
    if (P.dyn_sync && (s + 1 < nsteps || (multi && signal_mask))) {
        small_row_barrier(P, S, g, s);
        if (S.abort_flag) return false;
    }
    if (multi && signal_mask && t < 32 && ((signal_mask >> t) & 1u) && (!P.dyn_sync || blockIdx.x == 0)) {
        st_release_sys(&S.sym[t]->flags[g][fslot], (epoch << 8) | (uint64_t)(s + 1));
    }
    return true;
}

// KM: kSmallCommon or kSmallVar (variable pieces, P.small_var)
// AK: 0 = the 16-B path decided per step at run time, 1 = always 16-B, 2 = never (host-known)
template <int KM, int AK>
__global__ void __launch_bounds__(kSmallThreads, 1) mpxa_small_kernel(const __grid_constant__ ExecParams P) {
    constexpr bool VARK = KM == kSmallVar, LLK = KM == kSmallLL, LOC = KM == kSmallLocal || LLK;
    __shared__ SmallShared S;
    extern __shared__ __align__(16) char small_dyn[];
    CTA_STAMP(0);   // the program's moves, when they fit
    const int g = P.mode == 1 ? (int)blockIdx.y : P.my_gpu;
    const int t = threadIdx.x;
    const GpuProg prog = P.mode == 1 ? P.progs[g] : P.prog;
    const bool multi = P.G > 1;
    const bool cached = P.small_cache != 0;
    Move *smoves = reinterpret_cast<Move *>(small_dyn);
    // prologue (overlaps the previous kernel under PDL): step table and every move, once --
    // no descriptor round trip after the dependency wait
    const bool steps_smem = prog.nsteps <= kMaxStepsSmem;
    const bool ld_step = steps_smem && t < prog.nsteps;
    Step st_r;
    if (ld_step) st_r = prog.steps[t];
    if (LOC) {   // every move cached: resolve the moves to pointers once, here (destinations on
                 // peer GPUs keep their kind / rank: those bases arrive with the CTS)
        char *const work_g = P.small_swork ? small_dyn + swork_offset(P) : P.dc->work_base[g];
        for (int i = t; i < prog.nmoves; i += (int)blockDim.x) {
            const Move m = prog.moves[i];
            RMove r;
            r.src = local_base(P, g, work_g, m.src_kind, m.src_rank) + (uint64_t)m.src_off * P.unit;
            r.doff = (uint64_t)m.dst_off * P.unit;
            r.ll = m.dst_kind == BK_LL ? 1 : m.src_kind == BK_LL ? 2 : 0;
            r.dst_remote = !m.fanout && m.dst_kind != BK_LL && (int)m.dst_rank / P.R != g;
            r.dst_rank = m.dst_rank;
            r.dst = (m.fanout || r.dst_remote) ? nullptr
                    : r.ll == 1 ? reinterpret_cast<char *>(&P.dc->sym[m.dst_rank]->ll[0][g][m.dst_off])
                                : local_base(P, g, work_g, m.dst_kind, m.dst_rank) + r.doff;
            if (r.ll == 2) r.src = reinterpret_cast<const char *>(&P.dc->sym[g]->ll[0][m.src_rank][m.src_off]);
            r.n = (uint32_t)((uint64_t)m.len * P.unit);
            r.flow = m.flow;
            r.fanout = m.fanout;
            r.dst_kind = m.dst_kind;
            r.src_sm = P.small_swork && m.src_kind == BK_WORK;
            r.dst_sm = P.small_swork && m.dst_kind == BK_WORK && !m.fanout;
            reinterpret_cast<RMove *>(smoves)[i] = r;
        }
    } else if (cached) {
        for (int i = t; i < prog.nmoves; i += (int)blockDim.x) smoves[i] = prog.moves[i];
    }
    if (ld_step) S.steps[t] = StepInfo{st_r.move_begin, st_r.move_end - st_r.move_begin, st_r.signal_mask, st_r.wait_mask};
    if (t < P.G) {
        S.work_base[t] = (LOC && P.small_swork) ? small_dyn + swork_offset(P) : P.dc->work_base[t];
        S.sym[t] = P.dc->sym[t];
        S.recv_base[t] = P.mode == 0 ? P.recv
                         : P.mode == 1 ? (t == g ? P.recv + (uint64_t)t * P.R * P.recv_stride : nullptr)
                                       : (t == g ? P.recv : nullptr);
    }
    __syncthreads();
    griddep_wait();
    griddep_launch_dependents();
    if (t == 0) {
        S.cts_ok = 0;
        S.abort_flag = 0;
        S.epoch = multi ? *(volatile uint64_t *)&P.dc->epoch + 1 : 0;
        if (P.small_ll) {
            S.ll_seq = *(volatile uint64_t *)&P.dc->ll_seq + 1;
            S.ll_par = (S.ll_seq & 1) * sizeof(((SymRegion *)nullptr)->ll[0]);
        }
    }
    // rank bases known now: every rank's SEND / WORK row and the RECV rows of resolved GPUs
    fill_rank_bases(P, S, 0xffffffffu, true);
    __syncthreads();
    TRACE(0);
    const uint64_t epoch = S.epoch;
    if (multi && !P.small_ll) small_post_cts(P, S, g, epoch);
    const Move *mvs = cached ? smoves : prog.moves;
    const uint32_t ppm = (uint32_t)P.small_ppm;        // 16-byte pieces per move: power-of-two bound
    const uint32_t lg = 31u - (uint32_t)__clz((int)ppm);
    uint32_t prev_wait = 0;
    for (int s = 0; s < prog.nsteps; s++) {
        TRACE(11);
        StepInfo st;
        if (steps_smem) {
            st = S.steps[s];
        } else {
            const Step g_st = prog.steps[s];
            st = StepInfo{g_st.move_begin, g_st.move_end - g_st.move_begin, g_st.signal_mask, g_st.wait_mask};
        }
        const int fslot = P.dyn_sync ? 0 : (int)blockIdx.x;   // the row's flag in sync mode
        if (multi && !P.small_ll && !small_step_enter(P, S, g, s, prev_wait, st.signal_mask, epoch, fslot)) return;
        TRACE(13);
        // items = (move, 16-byte piece); thread t takes items t, t+T, ... four at a time:
        // all four loads in flight before the stores
        uint32_t items = (uint32_t)st.nm * ppm;
        uint32_t TT = gridDim.x * blockDim.x;
        uint32_t base0 = blockIdx.x * blockDim.x + t;
        const uint16_t *idx = nullptr;
        if (P.small_own) {          // this CTA's flows only (compacted move list), all its threads
            idx = reinterpret_cast<uint16_t *>(small_dyn + (size_t)P.small_cache * sizeof(Move));
            items = small_own_list(P, S, mvs + st.first, st.nm,
                                   reinterpret_cast<uint16_t *>(small_dyn + (size_t)P.small_cache * sizeof(Move)), LOC) *
                    ppm;
            TT = blockDim.x;
            base0 = t;
        }
        // 16-B fast path: the host vouched for every local offset / length / base, and the
        // recv bases of the peers written in this step arrived with their CTS
        // (AK != 0: the host knows the answer for the whole launch -- one copy path compiled)
        bool a16 = AK == 1 ? true : (AK == 2 || AK == 3) ? false : P.small_a16 != 0;
        const bool a8 = AK == 3;   // the host vouched for 8-B alignment of everything (not 16)
        if (AK == 0)
            for (int q = 0; q < P.G; q++)
                if (((st.signal_mask >> q) & 1u) && ((uintptr_t)S.recv_base[q] & 15)) a16 = false;
        TRACE(12);
        if (LLK) {   // sends (and local moves) first, then the receives
            const RMove *rm = reinterpret_cast<const RMove *>(smoves) + st.first;
            const int nrecv = (int)st.wait_mask, nsend = st.nm - nrecv;
            const uint32_t is = (uint32_t)nsend * ppm, ir = (uint32_t)nrecv * ppm;
            if (a16) {
                small_items_ll<true, false>(P, S, rm, is, lg, TT, base0, g);
                small_items_ll<true, true>(P, S, rm + nsend, ir, lg, TT, base0, g);
            } else {
                small_items_ll<false, false>(P, S, rm, is, lg, TT, base0, g);
                small_items_ll<false, true>(P, S, rm + nsend, ir, lg, TT, base0, g);
            }
        } else if (LOC) {
            const RMove *rm = reinterpret_cast<const RMove *>(smoves) + st.first;
            if (a16) small_items_loc<16>(P, S, rm, items, lg, TT, base0, idx);
            else if (a8) small_items_loc<8>(P, S, rm, items, lg, TT, base0, idx);
            else small_items_loc<0>(P, S, rm, items, lg, TT, base0, idx);
        } else if (VARK) {
            small_var_step(P, S, mvs, st.first, st.nm, a16, small_dyn);
        } else if (a16) {
            small_items<16>(P, S, mvs + st.first, items, lg, TT, base0, idx);
        } else {
            if (a8) small_items<8>(P, S, mvs + st.first, items, lg, TT, base0, idx);
            else small_items<0>(P, S, mvs + st.first, items, lg, TT, base0, idx);
        }
        TRACE(2);
        __syncthreads();
        TRACE(3 + (s < 7 ? s : 7));   // stamps 3..10: end of steps 0..7
        if (P.small_ll && S.abort_flag) return;   // a receive timed out (watchdog)
        if ((P.dyn_sync && (s + 1 < prog.nsteps || (multi && st.signal_mask))) || (multi && st.signal_mask))
            if (!small_step_exit(P, S, g, s, prog.nsteps, st.signal_mask, epoch, fslot)) return;
        TRACE(14);
        prev_wait = P.small_ll ? 0u : st.wait_mask;
    }
    if (multi || P.dyn_sync) small_finish(P, S, g, prog.nsteps, prev_wait, epoch);
    TRACE(15);
    CTA_STAMP(1);
}

// ------------------------------------------------------------------------------------
// Tiny launches: ONE step on ONE GPU (every rank local), every move cached -- the small
// single-GPU collectives (cfg1, small alltoall / allgather /
// alltoallv) -- as a kernel of its own.  The launch-latency floor of such calls is the
// instruction stream a cold SM runs (each launch lands on other SMs): no flags, CTS, step
// loop, rank table or path switches here, just resolve -> wait -> load -> store.
// ------------------------------------------------------------------------------------
struct TMove {
    const char *src;
    char *dst;          // non-fanout destination; fanout: offset inside every rank's buffer
    uint32_t n;         // bytes
    uint32_t fanout;    // 0, or 1 + the destination kind of a fan-out move
};
static_assert(sizeof(TMove) == 24, "TMove layout");

__device__ __forceinline__ char *tiny_base(const ExecParams &P, char *work, int kind, int rank) {
    return kind == BK_SEND ? (char *)P.send + (uint64_t)rank * P.send_stride
           : kind == BK_RECV ? P.recv + (uint64_t)rank * P.recv_stride
                             : work + (uint64_t)rank * P.work_stride;
}

template <int AW, int TB>
__global__ void __launch_bounds__(kSmallThreads, 1) mpxa_tiny_kernel(const __grid_constant__ ExecParams P) {
    extern __shared__ __align__(16) char tiny_dyn[];
    TMove *tm = reinterpret_cast<TMove *>(tiny_dyn);
    const int t = threadIdx.x;
    const int nm = P.prog.nmoves;
    // prologue (overlaps the previous kernel under PDL): resolve every move to pointers
    char *const work = P.dc->work_base[0];
    for (int i = t; i < nm; i += (int)blockDim.x) {
        const Move m = P.prog.moves[i];
        TMove r;
        r.src = tiny_base(P, work, m.src_kind, m.src_rank) + (uint64_t)m.src_off * P.unit;
        r.dst = m.fanout ? reinterpret_cast<char *>((uint64_t)m.dst_off * P.unit)
                         : tiny_base(P, work, m.dst_kind, m.dst_rank) + (uint64_t)m.dst_off * P.unit;
        r.n = (uint32_t)((uint64_t)m.len * P.unit);
        r.fanout = m.fanout ? 1u + m.dst_kind : 0u;
        tm[i] = r;
    }
    __syncthreads();
    griddep_wait();
    griddep_launch_dependents();
    const uint32_t ppm = (uint32_t)P.small_ppm, lg = 31u - (uint32_t)__clz((int)ppm), mask = ppm - 1u;
    const uint32_t items = (uint32_t)nm * ppm, TT = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + t; base < items; base += TT * TB) {
        PieceRegs<AW> R;
        const char *sp[TB];
#pragma unroll
        for (int k = 0; k < TB; k++) {
            sp[k] = nullptr;
            const uint32_t it = base + (uint32_t)k * TT;
            if (it >= items) continue;
            const TMove &m = tm[it >> lg];
            const uint32_t o = (it & mask) * 16;
            if (o >= m.n) continue;
            sp[k] = m.src + o;
            R.issue(k, sp[k], min(16u, m.n - o));
        }
#pragma unroll
        for (int k = 0; k < TB; k++) {
            if (!sp[k]) continue;
            const uint32_t it = base + (uint32_t)k * TT;
            const TMove &m = tm[it >> lg];
            const uint32_t o = (it & mask) * 16;
            const uint32_t len = min(16u, m.n - o);
            const uint4 val = R.value(k, sp[k]);
            if (!m.fanout) {
                store_piece<AW>(m.dst + o, val, len);
            } else {
                const uint64_t off = (uint64_t)(uintptr_t)m.dst + o;
#pragma unroll 1
                for (int r = 0; r < P.p; r++) store_piece<AW>(tiny_base(P, work, (int)m.fanout - 1, r) + off, val, len);
            }
        }
    }
}

// Tiny EAGER launches: one-step eager (LL) companion programs across GPUs (modes 1 and 2):
// every move resolved in the prologue; after the dependency wait this GPU's sends (payload
// words, each with the launch's flag, into the peers' staging) and local copies, then its
// receives (poll the words, copy the payload out).  The same word protocol as the general
// kernel's eager mode (small_items_ll), in a fraction of its code.
struct TLMove {
    const char *src;    // local source; receive: this GPU's staging (parity 0)
    char *dst;          // local destination; send: the peer's staging (parity 0); fan-out: offset
    uint32_t n;         // payload bytes (0: flag-only word)
    uint8_t ll;         // 0 local copy, 1 send, 2 receive
    uint8_t fan;        // 0, or 1 + destination kind: the payload goes to every rank of this GPU
    uint16_t pad;
};
static_assert(sizeof(TLMove) == 24, "TLMove layout");

__device__ __forceinline__ char *tl_base(const ExecParams &P, int g, char *work, int kind, int rank) {
    const uint64_t local = (uint64_t)(rank - g * P.R);
    if (kind == BK_SEND)
        return (char *)P.send + (P.mode == 2 ? 0 : (uint64_t)g * P.R * P.send_stride) + local * P.send_stride;
    if (kind == BK_RECV) return P.recv + (P.mode == 1 ? (uint64_t)g * P.R * P.recv_stride : 0) + local * P.recv_stride;
    return work + local * P.work_stride;
}

__global__ void __launch_bounds__(kSmallThreads, 1) mpxa_tiny_ll_kernel(const __grid_constant__ ExecParams P) {
    extern __shared__ __align__(16) char tiny_dyn[];
    TLMove *tm = reinterpret_cast<TLMove *>(tiny_dyn);
    const int t = threadIdx.x;
    const int g = P.mode == 1 ? (int)blockIdx.y : P.my_gpu;
    const GpuProg prog = P.mode == 1 ? P.progs[g] : P.prog;
    const int nm = prog.nmoves;
    char *const work = P.dc->work_base[g];
    for (int i = t; i < nm; i += (int)blockDim.x) {
        const Move m = prog.moves[i];
        TLMove r;
        r.ll = m.dst_kind == BK_LL ? 1 : m.src_kind == BK_LL ? 2 : 0;
        r.src = r.ll == 2 ? reinterpret_cast<const char *>(&P.dc->sym[g]->ll[0][m.src_rank][m.src_off])
                          : tl_base(P, g, work, m.src_kind, m.src_rank) + (uint64_t)m.src_off * P.unit;
        r.fan = m.fanout ? (uint8_t)(1 + m.dst_kind) : 0;
        r.dst = r.ll == 1 ? reinterpret_cast<char *>(&P.dc->sym[m.dst_rank]->ll[0][g][m.dst_off])
                : m.fanout ? reinterpret_cast<char *>((uint64_t)m.dst_off * P.unit)
                           : tl_base(P, g, work, m.dst_kind, m.dst_rank) + (uint64_t)m.dst_off * P.unit;
        r.n = (uint32_t)((uint64_t)m.len * P.unit);
        r.pad = 0;
        tm[i] = r;
    }
    const int nrecv = (int)prog.steps[0].wait_mask;   // receives are listed last
    __syncthreads();
    griddep_wait();
    griddep_launch_dependents();
    const uint64_t seq = *(volatile const uint64_t *)&P.dc->ll_seq + 1;
    const uint32_t f32 = (uint32_t)seq;                // (the flag word: low 32 bits of seq)
    const uint64_t par = (seq & 1) * sizeof(((SymRegion *)nullptr)->ll[0]);
    const uint32_t ppm = (uint32_t)P.small_ppm, lg = 31u - (uint32_t)__clz((int)ppm), mask = ppm - 1u;
    const uint32_t TT = gridDim.x * blockDim.x, b0 = blockIdx.x * blockDim.x + t;
    // phase 0: local copies and sends (no waiting); phase 1: receives
    for (int ph = 0; ph < 2; ph++) {
        const TLMove *mv = tm + (ph ? nm - nrecv : 0);
        const uint32_t items = (uint32_t)(ph ? nrecv : nm - nrecv) * ppm;
        for (uint32_t it = b0; it < items; it += TT) {
            const TLMove &m = mv[it >> lg];
            const uint32_t o = (it & mask) * 16;
            if (o >= m.n && !(m.ll && o == 0)) continue;
            const uint32_t len = m.n > o ? min(16u, m.n - o) : 0u;
            uint32_t d[4] = {0, 0, 0, 0};
            if (m.ll == 2) {                                // poll this piece's words
                const uint64_t *w = reinterpret_cast<const uint64_t *>(m.src + par) + o / 4;
                const uint32_t nw = len ? (len + 3) / 4 : 1;
                uint64_t t0 = 0;
                for (uint32_t j = 0; j < nw; j += 2) {
                    uint4 v = ld_ll_pair(w + j);
                    int spins = 0;
                    while (v.y != f32 || (j + 1 < nw && v.w != f32)) {
                        if (++spins > 64) {
                            __nanosleep(64);
                            if (!t0) t0 = globaltimer();
                            else if ((int64_t)(globaltimer() - t0) > P.timeout_ns) { atomicExch(P.err, 1); return; }
                        }
                        v = ld_ll_pair(w + j);
                    }
                    d[j] = v.x;
                    if (j + 1 < 4) d[j + 1] = v.z;
                }
            } else if (len) {                               // 4-byte words of the source piece
                const uintptr_t a = (uintptr_t)(m.src + o) & ~(uintptr_t)3;
                const uint32_t sh = 8u * (uint32_t)((uintptr_t)(m.src + o) & 3);
                const uint32_t *wp = (const uint32_t *)a;
                const uintptr_t end = (uintptr_t)(m.src + o) + len;
                uint32_t x[5];
#pragma unroll
                for (int q = 0; q < 5; q++) x[q] = (a + 4u * q < end) ? __ldcg(wp + q) : 0u;
#pragma unroll
                for (int q = 0; q < 4; q++) d[q] = __funnelshift_r(x[q], x[q + 1], sh);
            }
            if (m.ll == 1) {                                // send: words + flag to the peer
                uint64_t *w = reinterpret_cast<uint64_t *>(m.dst + par) + o / 4;
                const uint32_t nw = len ? (len + 3) / 4 : 1;
                for (uint32_t j = 0; j < nw; j += 2) {
                    if (j + 1 < nw) st_ll_pair(w + j, d[j], d[j + 1], f32);
                    else st_relaxed_sys(w + j, ((uint64_t)f32 << 32) | d[j]);
                }
                continue;
            }
            if (!len) continue;
            const uint4 val = make_uint4(d[0], d[1], d[2], d[3]);
            if (m.fan) {
                const uint64_t off = (uint64_t)(uintptr_t)m.dst + o;
#pragma unroll 1
                for (int r = g * P.R; r < (g + 1) * P.R; r++)
                    store_piece<0>(tl_base(P, g, work, m.fan - 1, r) + off, val, len);
            } else {
                store_piece<0>(m.dst + o, val, len);
            }
        }
    }
    // the launch's last CTA publishes the sequence number and the epoch (the general kernel's
    // eager launches advance both)
    __syncthreads();
    if (t == 0 && atom_acq_rel_gpu_add(&P.dc->done_ctas, 1u) == gridDim.x * gridDim.y - 1) {
        P.dc->done_ctas = 0;
        P.dc->epoch = *(volatile uint64_t *)&P.dc->epoch + 1;
        P.dc->ll_seq = seq;
    }
}

// Tiny MULTI-STEP launches: several steps on one GPU (Bruck, ring, hierarchical at small
// sizes), every move cached, in one CTA or in several CTAs that each own a set of flows --
// steps separated by __syncthreads only (a step reads what earlier steps of this CTA wrote).
template <int AW, int TB>
__global__ void __launch_bounds__(kSmallThreads, 1) mpxa_tiny_ms_kernel(const __grid_constant__ ExecParams P) {
    extern __shared__ __align__(16) char tiny_dyn[];
    __shared__ int2 st[kMaxStepsSmem];
    TMove *tm = reinterpret_cast<TMove *>(tiny_dyn);
    const int t = threadIdx.x;
    const int nm = P.prog.nmoves, ns = P.prog.nsteps;
    char *const work = P.dc->work_base[0];
    auto resolve = [&](const Move &m) {
        TMove r;
        r.src = tiny_base(P, work, m.src_kind, m.src_rank) + (uint64_t)m.src_off * P.unit;
        r.dst = m.fanout ? reinterpret_cast<char *>((uint64_t)m.dst_off * P.unit)
                         : tiny_base(P, work, m.dst_kind, m.dst_rank) + (uint64_t)m.dst_off * P.unit;
        r.n = (uint32_t)((uint64_t)m.len * P.unit);
        r.fanout = m.fanout ? 1u + m.dst_kind : 0u;
        return r;
    };
    if (P.small_own > 1) {
        // owned flows (several CTAs): this CTA keeps, step by step, only the moves of the flows
        // f with f % small_own == its index -- the same CTA moves a flow through every step,
        // so the steps still need no barrier but __syncthreads
        __shared__ uint32_t cnt;
        if (t == 0) cnt = 0;
        __syncthreads();
        for (int s = 0; s < ns; s++) {
            const Step sp = P.prog.steps[s];
            const uint32_t b = cnt;
            __syncthreads();
            for (int i = sp.move_begin + t; i < sp.move_end; i += (int)blockDim.x) {
                const Move m = P.prog.moves[i];
                if ((int)(m.flow % (uint32_t)P.small_own) == (int)blockIdx.x) tm[atomicAdd(&cnt, 1u)] = resolve(m);
            }
            __syncthreads();
            if (t == 0) st[s] = make_int2((int)b, (int)cnt);
        }
    } else {
        if (t < ns) {
            const Step s = P.prog.steps[t];
            st[t] = make_int2(s.move_begin, s.move_end);
        }
        for (int i = t; i < nm; i += (int)blockDim.x) tm[i] = resolve(P.prog.moves[i]);
    }
    __syncthreads();
    griddep_wait();
    griddep_launch_dependents();
    const uint32_t ppm = (uint32_t)P.small_ppm, lg = 31u - (uint32_t)__clz((int)ppm), mask = ppm - 1u;
    const uint32_t TT = blockDim.x;
    for (int s = 0; s < ns; s++) {
        const TMove *mv = tm + st[s].x;
        const uint32_t items = (uint32_t)(st[s].y - st[s].x) * ppm;
        for (uint32_t base = t; base < items; base += TT * TB) {
            PieceRegs<AW> R;
            const char *sp[TB];
#pragma unroll
            for (int k = 0; k < TB; k++) {
                sp[k] = nullptr;
                const uint32_t it = base + (uint32_t)k * TT;
                if (it >= items) continue;
                const TMove &m = mv[it >> lg];
                const uint32_t o = (it & mask) * 16;
                if (o >= m.n) continue;
                sp[k] = m.src + o;
                R.issue(k, sp[k], min(16u, m.n - o));
            }
#pragma unroll
            for (int k = 0; k < TB; k++) {
                if (!sp[k]) continue;
                const uint32_t it = base + (uint32_t)k * TT;
                const TMove &m = mv[it >> lg];
                const uint32_t o = (it & mask) * 16;
                const uint32_t len = min(16u, m.n - o);
                const uint4 val = R.value(k, sp[k]);
                if (!m.fanout) {
                    store_piece<AW>(m.dst + o, val, len);
                } else {
                    const uint64_t off = (uint64_t)(uintptr_t)m.dst + o;
#pragma unroll 1
                    for (int r = 0; r < P.p; r++) store_piece<AW>(tiny_base(P, work, (int)m.fanout - 1, r) + off, val, len);
                }
            }
        }
        __syncthreads();   // this step's writes before the next step's reads
    }
}

template <int AW>
static cudaError_t tiny_ms_attr() {
    static cudaError_t e = cudaFuncSetAttribute(mpxa_tiny_ms_kernel<AW, 1>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(kSmallMovesSmem * sizeof(TMove)));
    static cudaError_t f = cudaFuncSetAttribute(mpxa_tiny_ms_kernel<AW, kBatch>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(kSmallMovesSmem * sizeof(TMove)));
    return e != cudaSuccess ? e : f;
}
// every step's pieces (a CTA's share in the owned-flow mode) fit one pass of the block: the
// one-piece-per-thread build
template <int AW>
static cudaError_t launch_tiny_ms_aw(const ExecParams &P, int nC, int nt, size_t smem, bool pdl, cudaStream_t stream) {
    const cudaError_t a = tiny_ms_attr<AW>();
    if (a != cudaSuccess) return a;
    const uint64_t per = P.small_own > 1 ? (uint64_t)P.tiny_step_items * 2 / (uint64_t)nC : (uint64_t)P.tiny_step_items;
    const bool one = per <= (uint64_t)nt;
    return launch_kernel(one ? mpxa_tiny_ms_kernel<AW, 1> : mpxa_tiny_ms_kernel<AW, kBatch>, P, dim3(nC), dim3(nt),
                         smem, false, pdl, stream);
}


template <int AW>
static cudaError_t tiny_attr() {
    static cudaError_t e = cudaFuncSetAttribute(mpxa_tiny_kernel<AW, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(kSmallMovesSmem * sizeof(TMove)));
    static cudaError_t f = cudaFuncSetAttribute(mpxa_tiny_kernel<AW, kBatch>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(kSmallMovesSmem * sizeof(TMove)));
    return e != cudaSuccess ? e : f;
}
// one pass of the grid covers every piece: the one-piece-per-thread build (the shortest
// instruction stream -- tiny launches are instruction-fetch bound on cold SMs)
template <int AW>
static cudaError_t launch_tiny_aw(const ExecParams &P, int nC, int nt, size_t smem, bool pdl, cudaStream_t stream) {
    const cudaError_t a = tiny_attr<AW>();
    if (a != cudaSuccess) return a;
    const bool one = (uint64_t)P.prog.nmoves * (uint64_t)P.small_ppm <= (uint64_t)nC * (uint64_t)nt;
    return launch_kernel(one ? mpxa_tiny_kernel<AW, 1> : mpxa_tiny_kernel<AW, kBatch>, P, dim3(nC), dim3(nt), smem,
                         false, pdl, stream);
}

// Launch with the PDL attribute (pdl) and/or cooperatively.  cooperative = 1: the grid's CTAs
// wait on one another (emulated GPUs' CTA rows, per-step row barriers, peers across processes)
// and must be co-resident -- a cooperative launch guarantees it; 2: the same with PDL as well
// (accepted on sm_100a: tools/probes/coop_probe.cu, +0.1-0.25 us per launch over PDL alone).
// A cooperative launch the device cannot make co-resident falls back to the plain launch
// (grids are sized to the co-resident count, so this is a guard, not a path).
static cudaError_t launch_kernel(void (*kern)(ExecParams), const ExecParams &P, dim3 grid, dim3 block, size_t smem,
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

template <int KM, int AK>
static cudaError_t small_attr(size_t max_dyn) {
    static cudaError_t e = cudaFuncSetAttribute(mpxa_small_kernel<KM, AK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)max_dyn);
    return e;
}

template <int KM, int AK>
static cudaError_t launch_small_t(const ExecParams &P, size_t max_dyn, size_t smem, dim3 grid, int cooperative,
                                  bool pdl, cudaStream_t stream) {
    const cudaError_t a = small_attr<KM, AK>(max_dyn);
    if (a != cudaSuccess) return a;
    // P.small_threads: fewer threads for launches with few pieces per step -- the idle warps'
    // step bookkeeping competes with the working warp for issue slots (measured)
    const int nt = P.small_threads > 0 && !P.small_var ? P.small_threads : kSmallThreads;
    return launch_kernel(mpxa_small_kernel<KM, AK>, P, grid, dim3(nt), smem, cooperative, pdl, stream);
}

template <int KM>
static cudaError_t launch_small_km(const ExecParams &P, size_t max_dyn, size_t smem, dim3 grid, int cooperative,
                                   bool pdl, cudaStream_t stream) {
    // the 16-B decision is launch-wide unless peers' recv bases arrive at run time (mode 2)
    const int ak = P.mode == 2 ? 0 : (P.small_a16 ? 1 : (P.small_a8 ? 3 : 2));
    if (ak == 1) return launch_small_t<KM, 1>(P, max_dyn, smem, grid, cooperative, pdl, stream);
    if (ak == 3) return launch_small_t<KM, 3>(P, max_dyn, smem, grid, cooperative, pdl, stream);
    if (ak == 2) return launch_small_t<KM, 2>(P, max_dyn, smem, grid, cooperative, pdl, stream);
    return launch_small_t<KM, 0>(P, max_dyn, smem, grid, cooperative, pdl, stream);
}

cudaError_t launch_tiny_ms(const ExecParams &P, int nC, bool pdl, cudaStream_t stream) {
    const size_t smem = (size_t)P.prog.nmoves * sizeof(TMove);
    const int nt = P.small_threads > 0 ? P.small_threads : kSmallThreads;
    if (P.small_a16) return launch_tiny_ms_aw<16>(P, nC, nt, smem, pdl, stream);
    if (P.small_a8) return launch_tiny_ms_aw<8>(P, nC, nt, smem, pdl, stream);
    return launch_tiny_ms_aw<0>(P, nC, nt, smem, pdl, stream);
}

cudaError_t launch_tiny(const ExecParams &P, int nC, bool pdl, cudaStream_t stream) {
    const size_t smem = (size_t)P.prog.nmoves * sizeof(TMove);
    const int nt = P.small_threads > 0 ? P.small_threads : kSmallThreads;
    if (P.small_a16) return launch_tiny_aw<16>(P, nC, nt, smem, pdl, stream);
    if (P.small_a4) return launch_tiny_aw<4>(P, nC, nt, smem, pdl, stream);   // 4-byte words: no shifts
    if (P.small_a8) return launch_tiny_aw<8>(P, nC, nt, smem, pdl, stream);
    return launch_tiny_aw<0>(P, nC, nt, smem, pdl, stream);   // any alignment: words and funnel shifts
}

cudaError_t launch_tiny_ll(const ExecParams &P, int nC, int nG, int cooperative, bool pdl, cudaStream_t stream) {
    static cudaError_t a = cudaFuncSetAttribute(mpxa_tiny_ll_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(kSmallMovesSmem * sizeof(TLMove)));
    if (a != cudaSuccess) return a;
    int nmax = 0;   // the largest program of any GPU (emulated rows share the launch)
    if (P.mode == 1) {
        nmax = P.small_cache;
    } else {
        nmax = P.prog.nmoves;
    }
    const int nt = P.small_threads > 0 ? P.small_threads : kSmallThreads;
    return launch_kernel(mpxa_tiny_ll_kernel, P, dim3(nC, nG), dim3(nt), (size_t)nmax * sizeof(TLMove), cooperative,
                         pdl, stream);
}

cudaError_t launch_small(const ExecParams &P, int nC, int nG, int cooperative, bool pdl, cudaStream_t stream) {
    const dim3 grid(nC, nG);
    if (P.small_ll)
        return launch_small_km<kSmallLL>(P, kSmallMovesSmem * (sizeof(Move) + sizeof(uint16_t)),
                                         (size_t)P.small_cache * sizeof(Move), grid, cooperative, pdl, stream);
    if (!P.small_var && P.small_cache > 0 && P.p <= kRankTable)
        return launch_small_km<kSmallLocal>(P, kSmallMovesSmem * sizeof(Move) + kSmallWorkSmem,
                                            P.small_swork ? swork_offset(P) + (size_t)P.R * (size_t)P.work_stride
                                                          : (size_t)P.small_cache * sizeof(Move) +
                                                                (P.small_own ? (size_t)kSmallMovesSmem * sizeof(uint16_t)
                                                                             : 0),
                                            grid, cooperative, pdl, stream);
    if (P.small_var)
        return launch_small_km<kSmallVar>(P, kSmallMovesSmem * sizeof(Move) +
                                                 kSmallThreads * (sizeof(Move) + sizeof(uint32_t)),
                                          (size_t)P.small_cache * sizeof(Move) +
                                              (size_t)kSmallThreads * (sizeof(Move) + sizeof(uint32_t)),
                                          grid, cooperative, pdl, stream);
    return launch_small_km<kSmallCommon>(P, kSmallMovesSmem * (sizeof(Move) + sizeof(uint16_t)),
                                         (P.small_cache ? (size_t)P.small_cache * sizeof(Move) : 0) +
                                             (P.small_own ? (size_t)kSmallMovesSmem * sizeof(uint16_t) : 0),
                                         grid, cooperative, pdl, stream);
}

static cudaError_t exec_attr_once() {
    static cudaError_t e0 = cudaFuncSetAttribute(mpxa_exec_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kMaxDynSmem);
    static cudaError_t e1 = cudaFuncSetAttribute(mpxa_exec_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kMaxDynSmem);
    return e0 != cudaSuccess ? e0 : e1;
}

cudaError_t launch_exec(const ExecParams &P, int nC, int nG, int cooperative, bool pdl, cudaStream_t stream) {
    cudaError_t e = exec_attr_once();
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)P.stages * P.chunk;
    return launch_kernel(P.dyn_units ? mpxa_exec_kernel<true> : mpxa_exec_kernel<false>, P, dim3(nC, nG),
                         dim3(kThreads), smem, cooperative, pdl, stream);
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
    part_enter();
    if (threadIdx.x != 0) return;
    const int i = p0 + (int)(blockIdx.x / nct);
    const unsigned long long k = blockIdx.x % nct;
    const unsigned long long lo = k * chunk;
    const unsigned long long hi = lo + chunk < ch.part_bytes ? lo + chunk : ch.part_bytes;
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

int exec_max_ctas_per_sm(size_t dyn_smem) {
    if (exec_attr_once() != cudaSuccess) return 1;
    int n0 = 0, n1 = 0;   // both instantiations must fit the grids the host sizes
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n0, mpxa_exec_kernel<false>, kThreads, dyn_smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n1, mpxa_exec_kernel<true>, kThreads, dyn_smem);
    return std::min(n0, n1);
}

}  // namespace mpxa

#ifdef MPXA_TRACE
extern "C" int mpxa__cta_trace(uint64_t *out) {   // debug hook: [2][kMaxCtas] stamps; NULL resets
    if (!out) {
        static uint64_t zero[6][mpxa::kMaxCtas];
        return cudaMemcpyToSymbol(mpxa::g_cta_trace, zero, sizeof zero) == cudaSuccess ? 0 : 6;
    }
    return cudaMemcpyFromSymbol(out, mpxa::g_cta_trace, sizeof(mpxa::g_cta_trace)) == cudaSuccess ? 0 : 6;
}
#endif

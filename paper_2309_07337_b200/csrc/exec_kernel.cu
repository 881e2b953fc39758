// mpxa_exec_kernel (sm_100a) -- executes a collective PROGRAM (mpxa_internal.h): every step of
// pairwise / Bruck / ring / hierarchical alltoall(v) and allgather.
// Column-slice ownership: CTA c moves slice c of every move, so steps are separated by
// __syncthreads only; cross-GPU dependencies use per-(src GPU, CTA) release/acquire flags plus
// one clear-to-send (CTS) flag per GPU pair (A9).  Large single-step programs take pieces from
// device work queues (dynamic mode) through a TMA ring or per-warp rings.
#define MPXA_CTA_TRACE_OWNER
#include "kern_common.cuh"

namespace mpxa {

struct RingEntry {
    char *dst;          // non-fanout destination of the chunk
    uint64_t doff;      // fanout: byte offset inside every rank's dst_kind buffer
    uint32_t len;
    uint8_t fanout, dst_kind;
};

static_assert(kMoveTile <= kThreads, "prologue prefetch: one move per thread");

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

struct SmallJob {
    const char *src;
    char *dst;          // non-fanout destination (or first fan-out destination offset base)
    uint64_t doff;
    uint32_t n;
    uint8_t fanout, dst_kind, ro;
};

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

// Pre-wait L2 prefetch of the source of the pieces the grid takes first -- pieces c + k *
// gridDim.x, k < P.dyn_prefetch -- while the previous kernel finishes: a cache fill only (L2 is
// the device's point of coherence; the data is read after the wait), so the first loads after
// the wait hit L2 instead of queueing behind the whole grid's initial DRAM burst (measured,
// DESIGN §4 launch timeline).
__device__ __noinline__ void dyn_prefetch_first(const ExecParams &P, const ExecShared &S, int nm0) {
    const int t = threadIdx.x;
    if (t >= P.dyn_prefetch) return;
    const uint64_t U = (uint64_t)P.dyn_u;
    const uint32_t totA = S.pcA[nm0], tot = totA + S.pcB[nm0];
    const uint32_t u = blockIdx.x + (uint32_t)t * gridDim.x;
    if (u >= tot) return;
    const bool isA = u < totA;
    const uint32_t *pc = isA ? S.pcA : S.pcB;
    const uint32_t uu = isA ? u : u - totA;
    const int mi = find_move(pc, nm0, uu);
    const MovePlan mp = piece_plan(P, S, mi, (uint64_t)(uu - pc[mi]) * U, U);
    const uintptr_t a0 = (uintptr_t)mp.src & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)mp.src + mp.n + 15) & ~(uintptr_t)15;
    if (a1 > a0) prefetch_l2(a0, (uint32_t)(a1 - a0));
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
        // L2 prefetch of the source of the grid's first pieces (out of line: its code is only
        // fetched by launches that use it)
        if (P.dyn_prefetch) dyn_prefetch_first(P, S, nm0);
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

// The latency kernels (sm_100a): mpxa_small_kernel (short moves, items = (move, 16-B piece)
// pairs over all threads, moves cached in shared memory, eager / owned-flow / sync modes) and
// the tiny kernels for one-GPU and eager launches (mpxa_tiny_kernel, mpxa_tiny_ms_kernel,
// mpxa_tiny_ll_kernel), with their host launchers.
#include "kern_common.cuh"

namespace mpxa {

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

}  // namespace mpxa

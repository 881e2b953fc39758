// libmpxa host runtime: communicator, symmetric memory, program cache, launches, persistent
// requests, selector, and the C ABI of include/mpxa.h / include/mpxa_plan.h.
//
// Paper passages: MPIX_Comm_init / MPIX_Alltoallv (§2.1); persistent
// init/start/wait with setup paid once; default algorithm +
// every implementation selectable.  Argument contract and lifecycle errors
// follow SPEC.md:204-216, 239-247, 282-325 (interfaces only).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <string.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/mpxa.h"
#include "../../include/mpxa_plan.h"
#include "../../include/mpxa_device.cuh"
#include "mpxa_internal.h"
#include "plan.h"

namespace mpxa {
cudaError_t launch_exec(const ExecParams &P, int nC, int nG, int cooperative, bool pdl, cudaStream_t stream);
cudaError_t launch_small(const ExecParams &P, int nC, int nG, int cooperative, bool pdl, cudaStream_t stream);
cudaError_t launch_tiny(const ExecParams &P, int nC, bool pdl, cudaStream_t stream);
cudaError_t launch_tiny_ms(const ExecParams &P, int nC, bool pdl, cudaStream_t stream);
cudaError_t launch_tiny_ll(const ExecParams &P, int nC, int nG, int cooperative, bool pdl, cudaStream_t stream);
cudaError_t launch_counts(const int64_t *sc, int64_t *rc, int64_t *rd, int p, int r0, int nr,
                          cudaStream_t stream);
cudaError_t launch_scan(const int64_t *counts, int64_t *rc, int64_t *rd, int p, int nr,
                        cudaStream_t stream);
int exec_max_ctas_per_sm(size_t dyn_smem);
cudaError_t launch_part_start(bool sender, unsigned long long *cycle, unsigned long long *cts_remote,
                              cudaStream_t stream);
cudaError_t launch_part_pready(const mpxa_psend_dev_t &ch, int p0, int np, cudaStream_t stream);
cudaError_t launch_part_wait(const unsigned long long *flags, int lo, int hi, const unsigned long long *cycle,
                             int *err, long long timeout_ns, cudaStream_t stream);
}  // namespace mpxa

using namespace mpxa;

#define CK(x)                                                              \
    do {                                                                   \
        cudaError_t e_ = (x);                                              \
        if (e_ != cudaSuccess) {                                           \
            if (getenv("MPXA_DEBUG"))                                      \
                fprintf(stderr, "mpxa: %s failed: %s (%s:%d)\n", #x,       \
                        cudaGetErrorString(e_), __FILE__, __LINE__);       \
            return e_ == cudaErrorMemoryAllocation ? MPXA_ERR_NOMEM : MPXA_ERR_CUDA; \
        }                                                                  \
    } while (0)

namespace {

constexpr uint64_t kBytesPerCta = 65536;   // launch sizing target per CTA per step
constexpr uint64_t kSliceBytes = 16384;    // target column-slice length of the longest move
constexpr uint64_t kMovesPerCta = 1;       // moves per CTA (latency-bound regime: one each)
constexpr uint64_t kMinSlice = 2048;       // smallest slice worth a CTA when filling the GPU (= TMA min)
constexpr uint64_t kBigPerCta = 1u << 20;  // bytes per CTA per step above which the big TMA config wins
// small kernel: 16-B pieces per CTA per step -- about one per thread, so more CTAs share the
// bytes of a launch (measured, p = 8 one GPU: alltoall 1 / 4 / 16 KiB blocks 1.75 / 1.74 / 1.74
// -> 1.14 / 1.17 / 1.53 us going from 2048 to 256 pieces per CTA); fan-out pieces (allgather
// direct: one load, R stores) half of it (allgather 1 / 4 KiB 2.06 / 2.09 -> 1.48 / 1.51 us)
constexpr uint64_t kSmallItemsPerCta = 256;
constexpr uint64_t kSmallOneStepMove = 2u << 20;   // single-step programs: longest move ...
constexpr uint64_t kSmallOneStepVol = 32u << 20;   // ... and source bytes per GPU for the small kernel
                                                    // (re-measured after the small-kernel work:
                                                    // a2a p=8 512 KiB 13.5 -> 10.5 us, allgather
                                                    // p=4 2 MiB 11.4 -> 7.2 us; 64 MiB loses)
constexpr uint64_t kSmallSyncMove = 256u << 10;    // multi-step small launches on several CTAs:
constexpr uint64_t kSmallSyncVol = 8u << 20;       //   longest move, busiest step
// owned-flow mode: busiest step, and bytes per CTA (few flows -> few CTAs: allgathers).
// Measured on one B200: 8 MiB / 128 KiB (up from 2 MiB / 64 KiB) take p = 8 Bruck alltoall at
// 64 KiB blocks 12.1 -> 8.4 us, Bruck allgather 16 KiB 10.9 -> 7.9, ring allgather 64 KiB 17.8
// -> 15.8, p = 32 Bruck alltoall / allgather 4 KiB 29.0 / 68.8 -> 7.7 / 8.9 us; emulated GPUs
// (a row of CTAs per virtual GPU) keep the smaller limits -- there the larger ones lose up to 2x
// at 64-256 KiB
constexpr uint64_t kSmallOwnVol = 8u << 20;
constexpr uint64_t kSmallOwnPerCta = 128u << 10;
constexpr uint64_t kSmallOwnVolEmu = 2u << 20;
constexpr uint64_t kSmallOwnPerCtaEmu = 64u << 10;
constexpr uint64_t kSmallItemsOneCta = 2048;   // multi-step programs: largest step one CTA handles
constexpr uint64_t kDynMinMove = 128u << 10;   // dynamic mode: smallest average move (bytes) when
constexpr uint64_t kDynBigTotal = 128u << 20;  //   the busiest GPU moves this much, else ...
constexpr uint64_t kDynMinAvg = 512u << 10;    //   this average move (and kDynMinTotal)
constexpr uint64_t kDynMinTotal = 8u << 20;    // smallest per-GPU step volume
// multi-step dynamic mode (measured, p=8 on one B200): uniform blocks -- Bruck / hier alltoall,
// Bruck allgather gain 5-8 % from 4 MiB blocks (busiest step >= 128 MiB, >= 32 moves); below,
// or with few moves per step as in the ring, the per-step barrier costs more than the balance
// gains.  Uneven moves (alltoallv hier / Bruck-v, locality neighbor) gain 1.8-2.2x from 16 MiB.
constexpr uint64_t kDynSyncMin = 128u << 20;
constexpr int64_t kDynSyncMoves = 32;
constexpr uint64_t kDynSyncMinUneven = 16u << 20;
constexpr uint64_t kWringMinVol = 48u << 20;   // warp-ring mode: smallest busiest-GPU volume (96 MiB
                                               // before the constant-shift stores; measured since, cfg4:
                                               // mean 1 MiB (58 MiB) 25.9 / 29.5 -> 25.2 / 28.3 us with
                                               // the rings, mean 0.75 MiB (44 MiB) still LSU: 21.3 vs 22.9)
constexpr uint64_t kDynPiecesPerCta = 64;      // target queue pieces per CTA (measured: 16 -> 64 closes the tail)
constexpr uint64_t kDynMaxPiece = 512u << 10;  // largest piece (bytes)

// A program uploaded to device memory: [GpuProg x G][steps][moves].
struct DevProg {
    void *dmem = nullptr;
    size_t bytes = 0;
    Program host;
    int nsteps = 0;
    std::vector<GpuProg> gp;   // the [G] GpuProg table as uploaded (device pointers)
    int64_t max_gpu_moves = 0;      // most moves any GPU runs
    int64_t max_gpu_bytes_units = 0;  // single-step programs: most units any GPU moves (source side)
    int64_t dyn_tiles = 0;          // sum over steps of the most move tiles any GPU has in the step
    bool uniform_len = true;        // every move of the program has the same length
    bool fanout = false;            // some move writes every rank of a GPU (allgather direct)
    bool per_call = false;          // tables live in a ring slot (run_dynamic): no companions
    // Companion programs, built on first use and kept until the parent is freed: a CUDA graph
    // or a persistent request may hold device pointers into any of them, so a companion is
    // never replaced or freed while its parent lives (one entry per chop length / unit).
    //   var: small-kernel variable-piece companion -- long moves split into chop-unit moves
    //   ll:  eager (LL) companion per unit; a null entry marks the (program, unit) ineligible
    mutable std::map<int64_t, std::shared_ptr<DevProg>> var;
    mutable std::map<uint64_t, std::shared_ptr<DevProg>> ll;
};

// most companions one program keeps per kind (distinct units / chop lengths); beyond it the
// launch runs without one (the direct protocol / the plain piece decode -- same bytes)
constexpr size_t kMaxCompanions = 64;

// dynamic-mode eligibility facts of a program (DevProg::max_gpu_moves, max_gpu_bytes_units)
void prog_facts(DevProg &dp) {
    const Program &P = dp.host;
    dp.max_gpu_moves = 0;
    dp.max_gpu_bytes_units = 0;
    dp.dyn_tiles = 0;
    for (int s = 0; s < P.nsteps(); s++) {
        int64_t mx = 0;
        for (int g = 0; g < P.G; g++) mx = std::max<int64_t>(mx, P.steps[g][s].move_end - P.steps[g][s].move_begin);
        dp.dyn_tiles += std::max<int64_t>(1, (mx + kMoveTile - 1) / kMoveTile);
    }
    dp.uniform_len = true;
    dp.fanout = false;
    for (const auto &mv : P.moves)
        for (const Move &m : mv) {
            if (m.len != P.max_move) dp.uniform_len = false;
            if (m.fanout) dp.fanout = true;
        }
    for (const auto &mv : P.moves) {
        dp.max_gpu_moves = std::max<int64_t>(dp.max_gpu_moves, (int64_t)mv.size());
        int64_t u = 0;
        for (const Move &m : mv) u += m.len;
        dp.max_gpu_bytes_units = std::max(dp.max_gpu_bytes_units, u);
    }
}

size_t serialize(const Program &P, std::vector<char> &buf, uintptr_t dbase) {
    const int G = P.G;
    size_t off = sizeof(GpuProg) * G;
    std::vector<size_t> soff(G), moff(G), foff(G);
    for (int g = 0; g < G; g++) { soff[g] = off; off += sizeof(Step) * P.steps[g].size(); }
    for (int g = 0; g < G; g++) { moff[g] = off; off += sizeof(Move) * P.moves[g].size(); }
    for (int g = 0; g < G; g++) { foff[g] = off; off += sizeof(int32_t) * P.findex[g].size(); }
    buf.assign(off, 0);
    for (int g = 0; g < G; g++) {
        GpuProg gp{};
        gp.steps = (const Step *)(dbase + soff[g]);
        gp.moves = (const Move *)(dbase + moff[g]);
        gp.findex = (const int32_t *)(dbase + foff[g]);
        gp.nsteps = (int32_t)P.steps[g].size();
        gp.nmoves = (int32_t)P.moves[g].size();
        memcpy(buf.data() + sizeof(GpuProg) * g, &gp, sizeof gp);
        if (!P.steps[g].empty()) memcpy(buf.data() + soff[g], P.steps[g].data(), sizeof(Step) * P.steps[g].size());
        if (!P.moves[g].empty()) memcpy(buf.data() + moff[g], P.moves[g].data(), sizeof(Move) * P.moves[g].size());
        if (!P.findex[g].empty())
            memcpy(buf.data() + foff[g], P.findex[g].data(), sizeof(int32_t) * P.findex[g].size());
    }
    return off;
}

size_t serialized_size(const Program &P) {
    size_t n = sizeof(GpuProg) * P.G;
    for (int g = 0; g < P.G; g++)
        n += sizeof(Step) * P.steps[g].size() + sizeof(Move) * P.moves[g].size() +
             sizeof(int32_t) * P.findex[g].size();
    return n;
}

struct Window {
    uintptr_t base = 0;
    size_t size = 0;
};

struct SelEntry {
    int op, p, R;
    int G, g;            // GPUs of the comm and its group size (-1: any -- 5-field lines)
    uint64_t max_bytes;
    int algo;
};

// CTA decomposition: nS column slices per move x nF flow groups.  Depends
// only on the (global) program and the unit, so every process computes the same grid.
struct Grid {
    int nS = 1, nF = 1;
    bool big = false;   // TMA config: big (1 CTA / SM, 32 KiB stages) or mid
    int n() const { return nS * nF; }
};

// ring slot for per-call programs (v-ops)
struct Slot {
    void *dmem = nullptr;
    size_t cap = 0;
    char *pinned = nullptr;
    size_t pcap = 0;
    cudaEvent_t ev = nullptr;
    bool used = false;
};

}  // namespace

struct mpxa_comm_s {
    int nprocs = 1, proc = 0, R = 1, device = 0, g = 1;
    int G = 1;            // GPUs in programs (nprocs, or emulated GPUs)
    int p = 1;
    int Rg = 1;           // ranks per program GPU
    bool emulated = false;
    mpxa_allgather_fn boot = nullptr;
    void *ctx = nullptr;
    double timeout_s = 60.0;
    size_t heap0 = 0;                      // initial workspace heap per GPU (mpxa_init_args)
    int sm_count = 148, cap_ctas = 296;   // cap_ctas: mid TMA config (2 CTAs / SM)
    int cap_big = 148;                     // big TMA config (1 CTA / SM)
    int cap_small = 148;                   // small-message kernel (1 CTA / SM)
    int64_t var_chop = 32;                 // small kernel, variable pieces: longest move (bytes)
    int var_tiles = 4;                     // ... and warp tiles (32 moves) per CTA
    bool swork = true;                     // small kernel, one CTA on one GPU: WORK in shared memory
    int small_nt = 64;                     // small kernel block size for launches with few pieces
    bool ll = true;                        // eager (LL) mode for small multi-GPU launches
    uint64_t one_cta_items = kSmallItemsOneCta;  // MPXA_ONE_CTA_ITEMS (tuning)
    uint64_t small_items = kSmallItemsPerCta;    // MPXA_SMALL_ITEMS: 16-B pieces per small-kernel CTA
    uint64_t own_vol = 0;                        // MPXA_OWN_VOL / MPXA_OWN_PER_CTA: owned-flow mode
    uint64_t own_per_cta = 0;                    //   limits (busiest step; bytes per CTA); 0: default
    bool row_signal = true;                // MPXA_ROW_SIGNAL=0: executor steps signalled per (CTA, peer)
    bool hier_staged = false;              // MPXA_HIER_STAGED=1: hierarchical with group = GPU in its
                                           // literal three-step form instead of the fused one
    uint32_t last_path = 0;                // bits of the last launch's path (mpxa__last_launch)
    int64_t ll_max = 4 * kLLWords;         // eager: payload bytes per GPU pair, single-step launches
    int64_t ll_max_ms = 65536;             // ... multi-step launches
    int force_ns = 0, force_nf = 0;           // MPXA_NS / MPXA_NF overrides (tuning)
    int force_big = -1;                       // MPXA_TMA_BIG=0/1 override (tuning)
    bool force_exec = false;                  // MPXA_NO_SMALL=1: never use the small-message kernel
    bool pdl = true;                          // MPXA_NO_PDL=1: launches without programmatic serialization
    bool dyn = true;                          // MPXA_NO_DYN=1: static slices only (no work queue)
    int wring = 1;                            // warp-ring dynamic mode: 1 when moves may be misaligned,
                                              // MPXA_NO_WRING=1: never (LSU-register path), MPXA_WRING=2: always
    int dyn_pieces = (int)kDynPiecesPerCta;   // MPXA_DYN_PIECES: queue pieces per CTA (tuning)
    int wslack = 2;                           // MPXA_WSLACK: warp-ring stages kept out of the load window
    bool tiny = true;                         // MPXA_NO_TINY=1: small one-GPU launches in the general kernel
    bool tiny_even = true;                    // MPXA_TINY_EVEN=0: tiny-kernel blocks sized like the general kernel's
    uint64_t dyn_min_total = kDynMinTotal;    // MPXA_DYN_MIN: smallest busiest-GPU volume (tuning)
    int force_sync = -1;                      // MPXA_DYN_SYNC=0/1: force multi-step dynamic mode (tuning)
    bool small_sync = true;                   // MPXA_NO_SMALL_SYNC=1: multi-step small launches in one CTA
    uint64_t small_max1 = kSmallOneStepMove;  // MPXA_SMALL_MAX: longest move of one-step small launches
    uint64_t small_vol1 = kSmallOneStepVol;   // MPXA_SMALL_VOL: their source bytes per GPU (tuning)

    SymRegion *sym_local = nullptr;            // G regions when emulated, else 1
    SymRegion *sym_map[kMaxGpus] = {};
    char *work_local = nullptr;
    size_t work_bytes = 0;                     // per program GPU
    char *work_map[kMaxGpus] = {};
    int32_t *err_host = nullptr, *err_dev = nullptr;
    DevComm *dc = nullptr;                     // device-resident comm state (tables, epoch)
    DevComm dc_host;                           // host mirror of the tables
    std::vector<Window> windows;               // local registered windows (multi-process)
    std::vector<std::vector<char *>> win_map;  // [window][gpu] mapped bases

    uint64_t epoch = 0;
    uint64_t launches = 0;
    bool poisoned = false;
    mpxa_request_t active = nullptr;

    int user_algo[3] = {0, 0, 0};
    std::vector<SelEntry> selector;

    std::map<std::tuple<int, int, int, int>, std::shared_ptr<DevProg>> cache;  // (op,algo,stage,g)
    // one-shot alltoallv programs by (algo, global count / displacement matrices): repeated
    // calls with the same layout skip the build and the upload
    struct VEntry {
        int algo;
        std::vector<int64_t> C, SD, RD;
        std::shared_ptr<DevProg> prog;
        cudaEvent_t last = nullptr;      // recorded after the latest launch using prog
        uint64_t used = 0;
    };
    std::unordered_map<uint64_t, std::vector<VEntry>> vcache;
    uint64_t vcache_clock = 0;
    size_t vcache_n = 0;
    std::vector<Slot> ring;
    int ring_next = 0;
    int64_t *counts_tmp = nullptr;             // multi-process counts exchange staging
    size_t counts_tmp_bytes = 0;

    // f3 partitioned channels: a heap of 8-byte slots per process (cycle counters, CTS,
    // arrival flags, CTA counters), IPC-mapped by every process at the first match
    unsigned long long *part_local = nullptr;
    std::vector<unsigned long long *> part_map;   // [nprocs]
    std::vector<uint64_t> part_cursor;            // [nprocs] next free slot (same on every process)
    std::vector<mpxa_request_t> ppending;         // created, not yet matched (creation order)
    std::map<std::pair<int, std::string>, char *> ipc_opened;   // (proc, IPC handle bytes) -> mapped base
    cudaStream_t pquery = nullptr;                // private stream for Parrived host queries
};

struct mpxa_request_s {
    mpxa_comm_t comm = nullptr;
    int op = 0, algo = 0;
    bool active = false;
    std::shared_ptr<DevProg> prog;
    const char *send = nullptr;
    char *recv = nullptr;
    uint64_t unit = 0, send_stride = 0, recv_stride = 0;
    Grid grid;
    cudaEvent_t done = nullptr;
    cudaStream_t start_stream = nullptr;
    // f3 partitioned end (pkind 1 send, 2 receive)
    int pkind = 0, prank = 0, ppeer = 0, ptag = 0, nparts = 0;
    uint64_t part_bytes = 0;
    char *pbuf = nullptr;
    bool matched = false;
    uint64_t cycle = 0;                  // host mirror of this end's cycle
    std::vector<uint8_t> readied;        // sender: partitions readied this cycle (host calls)
    mpxa_psend_dev_t sdev{};             // sender device handle
    int peer_nparts = 0;                 // receiver: the sender's partitioning
    uint64_t peer_part_bytes = 0;
    unsigned long long *arr = nullptr;   // receiver: local arrival flags [peer_nparts]
    unsigned long long *mycycle = nullptr;    // this end's device cycle counter (local)
    unsigned long long *cts_remote = nullptr; // receiver: the sender's CTS slot (mapped)
};

struct mpxa_topo_s {
    mpxa_comm_t comm = nullptr;
    int p = 0;
    std::vector<int> indeg, src, outdeg, dst;   // global graph, rank-major edge lists
    std::vector<int> srcw, dstw;                // weights: stored, unused (SPEC.md decision)
    int64_t in0 = 0, out0 = 0;                  // this process's first in / out edge
    int64_t nin = 0, nout = 0;                  // this process's edge counts
};

namespace {

bool dtype_ok(size_t w) { return w == 1 || w == 2 || w == 4 || w == 8 || w == 16; }

// Host -> device copy of library tables that is COMPLETE on return.  A plain cudaMemcpy
// from pageable memory may return before its DMA has landed, and it runs on the legacy
// stream, which does not order the non-blocking streams our kernels are launched on; a
// table read by a kernel before the DMA lands would be stale.  So: an async copy on a
// private non-blocking stream of the current device, then a sync of that stream only (user
// streams are neither waited for nor blocked).  Tables are uploaded at init / first use,
// never inside a stream capture.
int h2d_complete(void *dst, const void *src, size_t n) {
    if (!n) return MPXA_SUCCESS;
    static std::mutex mu;
    static std::map<int, cudaStream_t> streams;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaStream_t st;
    {
        std::lock_guard<std::mutex> lk(mu);
        cudaStream_t &s = streams[dev];
        if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        st = s;
    }
    CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return MPXA_SUCCESS;
}

int bootstrap(mpxa_comm_t c, const void *in, void *out, size_t bytes) {
    if (c->nprocs == 1) { memcpy(out, in, bytes); return MPXA_SUCCESS; }
    if (!c->boot) return MPXA_ERR_ARG;
    return c->boot(in, out, bytes, c->ctx) == 0 ? MPXA_SUCCESS : MPXA_ERR_CUDA;
}

// all-gather variable-length byte strings (collective; two bootstrap rounds)
int allgather_var(mpxa_comm_t c, const void *mine, size_t n, std::vector<std::vector<char>> &out) {
    std::vector<uint64_t> sizes(c->nprocs);
    uint64_t n64 = n;
    int rc = bootstrap(c, &n64, sizes.data(), sizeof n64);
    if (rc) return rc;
    uint64_t mx = 0;
    for (uint64_t z : sizes) mx = std::max(mx, z);
    std::vector<char> pad(std::max<uint64_t>(mx, 1), 0), all((size_t)std::max<uint64_t>(mx, 1) * c->nprocs);
    if (n) memcpy(pad.data(), mine, n);
    rc = bootstrap(c, pad.data(), all.data(), pad.size());
    if (rc) return rc;
    out.assign(c->nprocs, {});
    for (int q = 0; q < c->nprocs; q++)
        out[q].assign(all.data() + (size_t)q * pad.size(), all.data() + (size_t)q * pad.size() + sizes[q]);
    return MPXA_SUCCESS;
}

template <typename T>
int allgather_concat(mpxa_comm_t c, const T *mine, size_t n, std::vector<T> &out) {
    std::vector<std::vector<char>> parts;
    int rc = allgather_var(c, mine, n * sizeof(T), parts);
    if (rc) return rc;
    out.clear();
    for (auto &b : parts) out.insert(out.end(), (const T *)b.data(), (const T *)(b.data() + b.size()));
    return MPXA_SUCCESS;
}

// ---- symmetric memory --------------------------------------------------------------

int ipc_exchange(mpxa_comm_t c, void *local, char **mapped) {
    // all-gather IPC handles of `local` and open every peer's
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, local));
    std::vector<cudaIpcMemHandle_t> all(c->nprocs);
    int rc = bootstrap(c, &h, all.data(), sizeof h);
    if (rc) return rc;
    for (int d = 0; d < c->nprocs; d++) {
        if (d == c->proc) { mapped[d] = (char *)local; continue; }
        void *ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, all[d], cudaIpcMemLazyEnablePeerAccess));
        mapped[d] = (char *)ptr;
    }
    return MPXA_SUCCESS;
}

// copy the host mirror of the device tables (work bases, symmetric regions, windows)
int upload_tables(mpxa_comm_t c) {
    if (!c->dc) return MPXA_SUCCESS;
    for (int g = 0; g < c->G; g++) {
        c->dc_host.work_base[g] = c->work_map[g];
        c->dc_host.sym[g] = c->sym_map[g];
    }
    return h2d_complete(c->dc, &c->dc_host, offsetof(DevComm, epoch));
}

int ensure_work(mpxa_comm_t c, size_t need_per_gpu) {
    if (need_per_gpu <= c->work_bytes) return MPXA_SUCCESS;
    size_t nb = std::max(need_per_gpu, c->work_bytes * 2);
    nb = (nb + 4095) & ~size_t(4095);
    CK(cudaDeviceSynchronize());   // growth is rare: retire work that may use the old heap
    if (c->nprocs > 1) {
        for (int d = 0; d < c->nprocs; d++)
            if (d != c->proc && c->work_map[d]) cudaIpcCloseMemHandle(c->work_map[d]);
    }
    if (c->work_local) cudaFree(c->work_local);
    c->work_local = nullptr;
    c->work_bytes = 0;
    size_t total = c->emulated ? nb * c->G : nb;
    CK(cudaMalloc((void **)&c->work_local, total));
    c->work_bytes = nb;
    if (c->nprocs > 1) {
        int rc = ipc_exchange(c, c->work_local, c->work_map);
        if (rc) return rc;
    } else {
        for (int g = 0; g < c->G; g++) c->work_map[g] = c->work_local + (size_t)g * nb;
    }
    return upload_tables(c);
}

// ---- selector -------------------------------------------------------------------------
int default_algo(mpxa_comm_t c, int op, size_t bytes) {
    if (c->user_algo[op]) return c->user_algo[op];
    // the measured table first (bench.py --write-selector); the rules below are fallbacks for
    // configurations no table row covers -- they were NOT measured on NVLink
    for (const SelEntry &e : c->selector)
        if (e.op == op && e.p == c->p && e.R == c->R && (e.G < 0 || e.G == c->G) && (e.g < 0 || e.g == c->g) &&
            bytes <= e.max_bytes)
            return e.algo;
    // SPEC.md:256 defaults when nothing was measured: pairwise (alltoall/v: its flags are
    // already one per GPU pair and CTA, so the hierarchical variant's fewer messages buy
    // nothing here).  Allgather: the direct (pairwise) exchange -- except across GPUs with
    // several ranks per GPU beyond the eager range, where direct fan-out sends every block to
    // each of a peer GPU's R ranks over NVLink and the hierarchical variant (groups = GPUs,
    // SURVEY §8 A10 "hier when R > 1") sends it once per GPU: R x fewer NVLink bytes.
    if (op == MPXA_OP_ALLGATHER && c->G > 1 && c->Rg > 1 && c->g == c->Rg &&
        (int64_t)bytes * c->Rg > c->ll_max)
        return A_HIER;
    return A_PAIRWISE;
}

bool algo_valid(int op, int algo) {
    if (op == MPXA_OP_ALLTOALL) return algo == A_PAIRWISE || algo == A_BRUCK || algo == A_HIER;
    if (op == MPXA_OP_ALLTOALLV) return algo == A_PAIRWISE || algo == A_HIER || algo == A_BRUCK;
    if (op == MPXA_OP_ALLGATHER) return algo == A_PAIRWISE || algo == A_BRUCK || algo == A_RING || algo == A_HIER;
    return false;
}

int upload_program(const Program &P, std::shared_ptr<DevProg> &out) {
    auto dp = std::make_shared<DevProg>();
    size_t n = serialized_size(P);
    CK(cudaMalloc(&dp->dmem, n ? n : 16));
    std::vector<char> buf;
    serialize(P, buf, (uintptr_t)dp->dmem);
    int rc = h2d_complete(dp->dmem, buf.data(), n);
    if (rc) { cudaFree(dp->dmem); return rc; }
    dp->gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + P.G);
    dp->bytes = n;
    dp->host = P;
    dp->nsteps = P.nsteps();
    prog_facts(*dp);
    out = dp;
    return MPXA_SUCCESS;
}

// The variable-piece companion of dp: moves longer than chop units become chop-unit moves
// (same flow, order and kinds), so tiles of kSmallThreads moves carry comparable piece
// counts and no CTA inherits a tile of whole long moves.  Small kernel only (no findex).
int var_program(const DevProg &dp, int64_t chop, const DevProg *&out) {
    out = nullptr;
    auto have = dp.var.find(chop);
    if (have != dp.var.end()) { out = have->second.get(); return MPXA_SUCCESS; }
    if (dp.var.size() >= kMaxCompanions) return MPXA_SUCCESS;
    {
        const Program &P = dp.host;
        Program Q;
        Q.p = P.p; Q.R = P.R; Q.G = P.G;
        Q.nflows = P.nflows;
        Q.work_units = P.work_units;
        Q.max_step_units = P.max_step_units;
        Q.signals = P.signals;
        Q.max_move = std::min<int64_t>(P.max_move, chop);
        Q.steps.resize(P.G);
        Q.moves.resize(P.G);
        Q.findex.assign(P.G, {});
        for (int g = 0; g < P.G; g++)
            for (const Step &st0 : P.steps[g]) {
                Step st = st0;
                st.move_begin = (int32_t)Q.moves[g].size();
                for (int32_t i = st0.move_begin; i < st0.move_end; i++) {
                    const Move &m = P.moves[g][i];
                    int64_t o = 0;
                    do {
                        Move x = m;
                        x.src_off += o;
                        x.dst_off += o;
                        x.len = std::min<int64_t>(chop, m.len - o);
                        Q.moves[g].push_back(x);
                        o += chop;
                    } while (o < m.len);
                }
                st.move_end = (int32_t)Q.moves[g].size();
                st.max_len = std::min<int64_t>(st.max_len, chop);
                st.flow_index = 0;
                st.dense_base = -1;
                Q.max_step_moves = std::max<int64_t>(Q.max_step_moves, st.move_end - st.move_begin);
                Q.steps[g].push_back(st);
            }
        auto v = std::shared_ptr<DevProg>(new DevProg, [](DevProg *d) {
            if (d->dmem) cudaFree(d->dmem);
            delete d;
        });
        size_t n = serialized_size(Q);
        CK(cudaMalloc(&v->dmem, n ? n : 16));
        std::vector<char> buf;
        serialize(Q, buf, (uintptr_t)v->dmem);
        int rc = h2d_complete(v->dmem, buf.data(), n);
        if (rc) return rc;
        v->gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + Q.G);
        v->bytes = n;
        v->host = std::move(Q);
        v->nsteps = v->host.nsteps();
        prog_facts(*v);
        dp.var[chop] = v;
        out = v.get();
    }
    return MPXA_SUCCESS;
}

// Upload a companion program (small kernel only: no flow index) as a self-freeing DevProg.
static int upload_companion(Program &&Q, std::shared_ptr<DevProg> &out) {
    auto v = std::shared_ptr<DevProg>(new DevProg, [](DevProg *d) {
        if (d->dmem) cudaFree(d->dmem);
        delete d;
    });
    size_t n = serialized_size(Q);
    CK(cudaMalloc(&v->dmem, n ? n : 16));
    std::vector<char> buf;
    serialize(Q, buf, (uintptr_t)v->dmem);
    int rc = h2d_complete(v->dmem, buf.data(), n);
    if (rc) return rc;
    v->gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + Q.G);
    v->bytes = n;
    v->host = std::move(Q);
    v->nsteps = v->host.nsteps();
    prog_facts(*v);
    out = v;
    return MPXA_SUCCESS;
}

// Eager (LL) companion of a program for one unit ("epoch-parity staging for
// eager mode"): every move whose destination is on a peer GPU d becomes
//   on its GPU g:  a SEND move to (BK_LL, d, word offset w) -- the payload as 4-byte words,
//                  each stored with the launch's flag in one 8-byte word into d's staging;
//   on GPU d:      a RECEIVE move (BK_LL, g, w) -> the original destination, which polls
//                  the words until they carry the flag.
// Fan-out moves (allgather direct) keep a local fan-out (fanout = 2: this GPU's ranks) and
// send one stream per peer GPU, which the peer fans out to its own ranks.  Word offsets run
// per (g, d) pair across all steps of the launch; a pair without data still exchanges one
// flag word, so every GPU hears from every peer in every eager launch -- which is what makes
// the two staging parities safe to alternate.  In each step the receive moves come last
// (Step::wait_mask = their number): a CTA issues all its sends before it polls.
// Returns false when a pair needs more than kLLWords words or a GPU more moves than the
// small kernel caches.
static bool build_ll(const Program &P, uint64_t unit, int R, Program &Q, int64_t max_words = kLLWords) {
    const int G = P.G, ns = P.nsteps();
    Q = Program();
    Q.p = P.p; Q.R = P.R; Q.G = G;
    Q.nflows = P.nflows;
    Q.work_units = P.work_units;
    Q.max_step_units = P.max_step_units;
    Q.max_move = P.max_move;
    Q.signals = 0;
    Q.steps.assign(G, {});
    Q.moves.assign(G, {});
    Q.findex.assign(G, {});
    std::vector<int64_t> wc((size_t)G * G, 0);
    auto words = [&](const Move &m) { return std::max<int64_t>(1, (int64_t)((m.len * unit + 3) / 4)); };
    for (int s = 0; s < ns; s++) {
        std::vector<std::vector<Move>> out(G), in(G);
        for (int g = 0; g < G; g++) {
            const Step &st = P.steps[g][s];
            for (int32_t i = st.move_begin; i < st.move_end; i++) {
                const Move &m = P.moves[g][i];
                if (m.fanout) {
                    Move x = m;
                    x.fanout = 2;
                    out[g].push_back(x);
                }
                for (int d = 0; d < G; d++) {
                    if (d == g) continue;
                    if (!m.fanout && (int)m.dst_rank / R != d) continue;
                    int64_t &w0 = wc[(size_t)g * G + d];
                    w0 += w0 & 1;   // even word offsets: 16-byte aligned pairs of words
                    Move snd = m, rcv = m;
                    snd.fanout = 0;
                    snd.dst_kind = BK_LL;
                    snd.dst_rank = (uint16_t)d;
                    snd.dst_off = wc[(size_t)g * G + d];
                    rcv.fanout = m.fanout ? 2 : 0;
                    rcv.src_kind = BK_LL;
                    rcv.src_rank = (uint16_t)g;
                    rcv.src_off = wc[(size_t)g * G + d];
                    wc[(size_t)g * G + d] += words(m);
                    out[g].push_back(snd);
                    in[d].push_back(rcv);
                }
                if (!m.fanout && (int)m.dst_rank / R == g) out[g].push_back(m);
            }
        }
        if (s == 0)   // flag-only words for pairs without data in the whole launch
            for (int g = 0; g < G; g++)
                for (int d = 0; d < G; d++) {
                    if (d == g) continue;
                    bool any = false;
                    for (int s2 = 0; s2 < ns && !any; s2++) {
                        const Step &st = P.steps[g][s2];
                        for (int32_t i = st.move_begin; i < st.move_end && !any; i++) {
                            const Move &m = P.moves[g][i];
                            any = m.fanout || (int)m.dst_rank / R == d;
                        }
                    }
                    if (any) continue;
                    Move snd{}, rcv{};
                    snd.src_kind = BK_SEND;
                    snd.src_rank = (uint16_t)(g * R);
                    snd.dst_kind = BK_LL;
                    snd.dst_rank = (uint16_t)d;
                    rcv.src_kind = BK_LL;
                    rcv.src_rank = (uint16_t)g;
                    rcv.dst_kind = BK_RECV;
                    rcv.dst_rank = (uint16_t)(d * R);
                    wc[(size_t)g * G + d] = 1;
                    out[g].push_back(snd);
                    in[d].push_back(rcv);
                }
        for (int g = 0; g < G; g++) {
            Step st = P.steps[g][s];
            st.move_begin = (int32_t)Q.moves[g].size();
            for (const Move &m : out[g]) Q.moves[g].push_back(m);
            for (const Move &m : in[g]) Q.moves[g].push_back(m);
            st.move_end = (int32_t)Q.moves[g].size();
            st.signal_mask = 0;
            st.wait_mask = (uint32_t)in[g].size();
            st.flow_index = 0;
            st.dense_base = -1;
            Q.max_step_moves = std::max<int64_t>(Q.max_step_moves, st.move_end - st.move_begin);
            Q.steps[g].push_back(st);
        }
    }
    for (int64_t w : wc)
        if (w > std::min<int64_t>(max_words, kLLWords)) return false;
    for (int g = 0; g < G; g++)
        if (Q.moves[g].size() > (size_t)kSmallMovesSmem) return false;
    return true;
}

// The eager companion of dp for `unit`, built on first use (never inside a stream capture:
// the upload is synchronous).  nullptr when ineligible or not available.
static const DevProg *ll_program(mpxa_comm_t c, const DevProg &dp, uint64_t unit, cudaStream_t stream) {
    auto have = dp.ll.find(unit);
    if (have != dp.ll.end()) return have->second.get();
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (dp.per_call || cudaStreamIsCapturing(stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return nullptr;
    if (dp.ll.size() >= kMaxCompanions) return nullptr;
    std::shared_ptr<DevProg> &slot = dp.ll[unit];   // null = ineligible (kept: decided once)
    Program Q;
    // measured (4 emulated GPUs, p = 4 / 8): eager wins up to the full 128 KiB staging per
    // GPU pair for single-step launches (pairwise alltoall 64 KiB pairs 16.0 -> 10.2 us; the
    // direct protocol's CTS + two system-scope releases cost more than eager's 2x bytes);
    // multi-step ones pay the 2x bytes and word stores in every step; re-measured after the
    // executor's per-GPU signalling: eager still wins at 64 KiB per pair (ring allgather 4 KiB
    // blocks 37.5 -> 19.7 us, Bruck alltoall 2 KiB 24.5 -> 16.2 us on 4 emulated GPUs)
    const int64_t max_words = (dp.nsteps > 1 ? c->ll_max_ms : c->ll_max) / 4;
    if (!build_ll(dp.host, unit, c->Rg, Q, max_words)) return nullptr;
    std::shared_ptr<DevProg> up;
    if (upload_companion(std::move(Q), up) != MPXA_SUCCESS) return nullptr;
    slot = up;
    return slot.get();
}

// Persistent *_init: build the eager companion now (collective, outside any stream capture),
// so a first start() inside a CUDA-graph capture already runs eager, the same in every process.
static void prebuild_companions(mpxa_comm_t c, const DevProg &dp, uint64_t unit) {
    if (c->ll && c->G > 1 && c->p <= kRankTable) (void)ll_program(c, dp, unit, (cudaStream_t)0);
}

int cached_uniform(mpxa_comm_t c, int op, int algo, int stage, std::shared_ptr<DevProg> &out) {
    auto key = std::make_tuple(op, algo, stage, c->g);
    auto it = c->cache.find(key);
    if (it != c->cache.end()) { out = it->second; return MPXA_SUCCESS; }
    Program P;
    bool ok = op == MPXA_OP_ALLTOALL ? build_alltoall(P, algo, c->p, c->Rg, c->G, c->g, stage, c->hier_staged)
                                     : build_allgather(P, algo, c->p, c->Rg, c->G, stage, c->g);
    if (!ok) return MPXA_ERR_ALGO;
    int rc = upload_program(P, out);
    if (rc) return rc;
    c->cache[key] = out;
    return MPXA_SUCCESS;
}


uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

Grid choose_grid(mpxa_comm_t c, const Program &P, uint64_t unit) {
    const uint64_t L = (uint64_t)P.max_move * unit;          // longest move
    const uint64_t T = (uint64_t)P.max_step_units * unit;    // busiest step of one GPU
    Grid gr;
    // large steps stream through fewer, fatter pipelines; the rest through more CTAs
    gr.big = c->force_big >= 0 ? c->force_big > 0 : T / (uint64_t)c->cap_big >= kBigPerCta;
    const uint64_t cap = (uint64_t)(gr.big ? c->cap_big : c->cap_ctas);
    uint64_t nS = std::min<uint64_t>(cap, std::max<uint64_t>(1, cdiv(L, kSliceBytes)));
    uint64_t nF_bw = cdiv(T, nS * kBytesPerCta);              // enough CTAs for bandwidth
    uint64_t nF_lat = cdiv((uint64_t)P.max_step_moves, kMovesPerCta);  // ~1 move per LSU warp
    uint64_t nF = std::max<uint64_t>(1, std::max(nF_bw, nF_lat));
    nF = std::min<uint64_t>(nF, std::max<uint64_t>(1, cap / nS));
    nF = std::min<uint64_t>(nF, (uint64_t)P.nflows);
    if (c->force_ns > 0) nS = (uint64_t)c->force_ns;
    if (c->force_nf > 0) nF = std::min<uint64_t>((uint64_t)c->force_nf, (uint64_t)P.nflows);
    while (nS * nF > (uint64_t)kMaxCtas || nS * nF > cap) {
        if (nF > 1) nF--;
        else nS--;
    }
    // fill the machine: widen the slices' count to use every resident CTA slot when the
    // slices stay >= kMinSlice bytes
    if (c->force_ns <= 0 && nF >= 1) {
        uint64_t wide = cap / nF;
        if (wide > nS && L / wide >= kMinSlice) nS = wide;
        else if (wide > nS && L / kMinSlice > nS) nS = std::min<uint64_t>(wide, L / kMinSlice);
    }
    gr.nS = (int)std::max<uint64_t>(1, nS);
    gr.nF = (int)std::max<uint64_t>(1, nF);
    return gr;
}

// Fill launch parameters for a program on this comm.
int make_params(mpxa_comm_t c, ExecParams &E, const DevProg &dp, const char *send, char *recv,
                uint64_t unit, uint64_t send_stride, uint64_t recv_stride) {
    memset(&E, 0, sizeof E);
    E.progs = (const GpuProg *)dp.dmem;
    if (!c->emulated) E.prog = dp.gp[c->nprocs > 1 ? c->proc : 0];
    E.dc = c->dc;
    E.send = send;
    E.recv = recv;
    E.unit = unit;
    E.send_stride = send_stride;
    E.recv_stride = recv_stride;
    E.work_stride = (uint64_t)dp.host.work_units * unit;
    E.err = c->err_dev;
    E.timeout_ns = (int64_t)(c->timeout_s * 1e9);
    E.G = c->G;
    E.R = c->Rg;
    E.p = c->p;
    E.nflows = dp.host.nflows;
    E.my_gpu = c->emulated ? -1 : (c->nprocs > 1 ? c->proc : 0);
    E.mode = c->emulated ? 1 : (c->nprocs > 1 ? 2 : 0);
    // step 0 dense on EVERY GPU with one base flow and count (single program per launch
    // in modes 0 / 2; emulated launches need them equal across the virtual GPUs)
    E.d0_base = -1;
    if (dp.nsteps > 0) {
        const int g0 = c->emulated ? 0 : (c->nprocs > 1 ? c->proc : 0);
        const Step &s0 = dp.host.steps[g0][0];
        bool ok = s0.dense_base >= 0;
        if (c->emulated)
            for (int g = 1; g < c->G && ok; g++) {
                const Step &o = dp.host.steps[g][0];
                ok = o.dense_base == s0.dense_base && o.move_end == s0.move_end;
            }
        if (ok) { E.d0_base = s0.dense_base; E.d0_n = s0.move_end - s0.move_begin; }
    }
    if (c->nprocs > 1) {
        // remote recv bases are resolved on the device from the CTS message (window + offset)
        uintptr_t r = (uintptr_t)recv;
        int wi = -1;
        for (size_t w = 0; w < c->windows.size(); w++)
            if (r >= c->windows[w].base && r < c->windows[w].base + c->windows[w].size) { wi = (int)w; break; }
        if (wi < 0) return MPXA_ERR_UNREGISTERED;
        E.recv_win = (uint64_t)wi;
        E.recv_off = r - c->windows[wi].base;
    }
    return MPXA_SUCCESS;
}

// Cooperative level of a launch (kern_common.cuh launch_kernel): CTAs that wait on one another must
// be co-resident.  Emulated GPUs: cooperative (their CTA rows exchange flags; launches as in
// round 1, no PDL).  Across processes every CTA may wait on a peer GPU's CTAs, which wait on
// this grid's: cooperative + PDL, so no CTA spins while another of its grid is not scheduled
// (another stream's kernel holding SMs).  One GPU: only launches with per-step row barriers
// (barriers: several steps over several CTAs, not owned-flow).
static int coop_level(mpxa_comm_t c, bool barriers) {
    if (c->emulated) return 1;
    return (c->nprocs > 1 || barriers) ? 2 : 0;
}

// pdl: the launch may overlap the previous kernel's tail (the kernel waits on
// griddepcontrol before touching anything that kernel wrote).  Off for per-call programs,
// whose tables arrive by a cudaMemcpyAsync right before the launch.
int run_program(mpxa_comm_t c, const DevProg &dp, const char *send, char *recv, uint64_t unit,
                uint64_t send_stride, uint64_t recv_stride, cudaStream_t stream, const Grid *grid = nullptr,
                bool pdl = true) {
    if (c->poisoned) return MPXA_ERR_TIMEOUT;
    if (dp.nsteps == 0) return MPXA_SUCCESS;
    size_t need = (size_t)dp.host.work_units * unit * c->Rg;
    int rc = ensure_work(c, need);
    if (rc) return rc;
    ExecParams E;
    rc = make_params(c, E, dp, send, recv, unit, send_stride, recv_stride);
    if (rc) return rc;
    const Grid gr = grid ? *grid : choose_grid(c, dp.host, unit);
    E.nS = gr.nS;
    E.nF = gr.nF;
    const TmaConfig tc = gr.big ? kTmaBig : kTmaMid;
    E.stages = tc.stages;
    E.chunk = tc.chunk;
    E.ahead = tc.ahead;
    ++c->epoch;   // host mirror only; the kernels keep the authoritative epoch in DevComm
    cudaError_t e;
    int coop = 0;   // cooperative level of the launch (coop_level)
    bool tiny = false;
    const uint64_t maxmove = (uint64_t)dp.host.max_move * unit;
    uint64_t ppm = 1;   // 16-B pieces per move, rounded up to a power of two (shift decode)
    while (ppm * 16 < maxmove) ppm <<= 1;
    // pieces per step, fan-out stores counted per destination (max_step_units counts them)
    const uint64_t slots = std::max<uint64_t>((uint64_t)dp.host.max_step_moves,
                                              (uint64_t)dp.host.max_step_units / std::max<int64_t>(1, dp.host.max_move)) * ppm;
    // moves of very different lengths (e.g. element runs next to whole blocks): max-move slots
    // per move are mostly empty -- the small kernel then counts pieces exactly per tile of moves
    const uint64_t exact = (uint64_t)dp.host.max_step_units * unit / 16 + (uint64_t)dp.host.max_step_moves;
    const bool var = !dp.uniform_len && exact * 4 < slots;
    const uint64_t items = var ? exact : slots;
    const bool one_step = dp.nsteps == 1;
    // Small-message kernel: multi-step programs with short moves and a step small enough for
    // one CTA; single-step programs (any number of CTAs) up to 2 MiB moves and 32 MiB of
    // source data per GPU -- measured on one B200: its LSU pieces beat the TMA executor's
    // fixed costs there (alltoall 64 KiB blocks 5.3 -> 3.8 us, allgather 1 MiB 17.9 -> 13.8 us,
    // alltoallv cfg4 64 KiB mean 9.2 -> 5.2 us); beyond, the executor streams better.
    const uint64_t src_vol = (uint64_t)dp.max_gpu_bytes_units * unit;
    // multi-step programs too large for one CTA but small in volume: several CTAs with a
    // barrier between steps (sync mode)
    const uint64_t step_vol = (uint64_t)dp.host.max_step_units * unit;
    // (measured: it wins where the static executor is poorly balanced -- uneven moves, or few
    // flows to spread over CTAs as in the allgathers; uniform alltoalls keep the barrier-free
    // static executor)
    const uint64_t per_cta = dp.fanout ? std::max<uint64_t>(32, c->small_items / 2) : c->small_items;
    const uint64_t n_own = std::max<uint64_t>(1, std::min<uint64_t>(std::min<uint64_t>(cdiv(items, per_cta),
                                                                                          (uint64_t)dp.host.nflows),
                                                                     (uint64_t)c->cap_small));
    const uint64_t own_vol = c->own_vol ? c->own_vol : c->emulated ? kSmallOwnVolEmu : kSmallOwnVol;
    const uint64_t own_per_cta = c->own_per_cta ? c->own_per_cta : c->emulated ? kSmallOwnPerCtaEmu : kSmallOwnPerCta;
    const bool own_ok = dp.uniform_len && step_vol <= own_vol && step_vol / n_own <= own_per_cta;
    const bool small_sync = !one_step && items > c->one_cta_items && maxmove <= kSmallSyncMove &&
                            step_vol <= kSmallSyncVol && c->small_sync &&
                            (!own_ok || dp.max_gpu_moves > kSmallMovesSmem) &&
                            (!dp.uniform_len || dp.host.nflows < 32 || dp.max_gpu_moves > kSmallMovesSmem);
    // uniform multi-step programs (flows of equal size, moved whole in every step): several
    // CTAs, each owning the flows f % nC == c through all steps -- no barrier needed
    // (measured, p=8: Bruck alltoall 4 KiB 13.9 -> 10.8 us, hier 9.8 -> 8.6 us at 16 KiB; from
    // 64 KiB blocks the TMA executor is faster again)
    const bool small_own = !one_step && !small_sync && items > c->one_cta_items && maxmove <= kSmallSyncMove &&
                           own_ok && c->small_sync && dp.max_gpu_moves <= kSmallMovesSmem;
    // (emulated GPUs share the SMs: a virtual GPU's small-kernel row has 1/G of them, and its
    // LSU pieces lose to the executor's TMA on long moves sooner -- measured: f1 halo, 2 MiB
    // moves on 4 emulated GPUs, 47 -> 32 us with the executor; cfg5's 64-256 KiB moves stay
    // 3x faster in the small kernel)
    const uint64_t max1 = c->emulated ? std::min<uint64_t>(c->small_max1, 1u << 20) : c->small_max1;
    const bool small = !c->force_exec &&
                       (one_step ? (maxmove <= max1 && src_vol <= c->small_vol1)
                                 : ((maxmove <= kSmallKernelMax && items <= c->one_cta_items) || small_sync ||
                                    small_own));
    if (small) {
        E.nS = E.nF = 1;
        E.small_a16 = unit % 16 == 0 && (uintptr_t)send % 16 == 0 && (uintptr_t)recv % 16 == 0 &&
                      send_stride % 16 == 0 && recv_stride % 16 == 0 && E.work_stride % 16 == 0;
        // int64 / double payloads: 8-byte words instead of 4-byte words and funnel shifts (eager
        // launches keep their own 4-byte word streams; a per-process choice -- no protocol
        // consequence across processes)
        E.small_a8 = !E.small_a16 && unit % 8 == 0 && (uintptr_t)send % 8 == 0 && (uintptr_t)recv % 8 == 0 &&
                     send_stride % 8 == 0 && recv_stride % 8 == 0 && E.work_stride % 8 == 0;
        E.small_a4 = !E.small_a16 && !E.small_a8 && unit % 4 == 0 && (uintptr_t)send % 4 == 0 &&
                     (uintptr_t)recv % 4 == 0 && send_stride % 4 == 0 && recv_stride % 4 == 0 &&
                     E.work_stride % 4 == 0;
        E.small_ppm = (int32_t)ppm;
        const DevProg *sp = &dp;
        // variable pieces: long moves split (companion program) unless the tables are per-call
        // or the stream is being captured (the companion's upload is synchronous)
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        const int64_t chop = std::max<int64_t>(1, c->var_chop / (int64_t)unit);
        if (var && !dp.per_call && c->var_chop > 0 && (uint64_t)dp.host.max_move * unit > (uint64_t)c->var_chop &&
            (dp.var.count(chop) ||
             (cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone))) {
            const DevProg *vp = nullptr;
            rc = var_program(dp, chop, vp);
            if (rc) return rc;
            if (vp) {
                sp = vp;
                E.progs = (const GpuProg *)sp->dmem;
                if (!c->emulated) E.prog = sp->gp[c->nprocs > 1 ? c->proc : 0];
            }
        }
        // eager (LL) mode: several GPUs, small launches -- the payload travels with its flags,
        // no CTS, no system-scope release (build_ll)
        if (c->ll && c->G > 1 && !var && c->p <= kRankTable) {
            if (const DevProg *lp = ll_program(c, dp, unit, stream)) {
                sp = lp;
                E.small_ll = 1;
                E.progs = (const GpuProg *)sp->dmem;
                if (!c->emulated) E.prog = sp->gp[c->nprocs > 1 ? c->proc : 0];
            }
        }
        size_t nmoves_g = 0;
        for (const auto &mv : sp->host.moves) nmoves_g = std::max(nmoves_g, mv.size());
        E.small_cache = nmoves_g <= (size_t)kSmallMovesSmem ? (int32_t)nmoves_g : 0;
        int nC = (one_step || small_sync || small_own)
                     ? (int)std::min<uint64_t>(cdiv(items, per_cta), (uint64_t)c->cap_small) : 1;
        if (small_own) nC = std::min<int>(nC, dp.host.nflows);
        E.dyn_sync = small_sync && nC > 1;
        E.small_own = small_own && nC > 1 ? nC : 0;
        if (E.small_ll && E.small_own) {   // eager steps take every piece of the step (no flow
            E.small_own = 0;               // ownership): CTAs meet at the row barrier instead
            E.dyn_sync = 1;
        }
        E.small_var = var && !E.small_own;
        if (E.small_var) {   // warp tiles of 32 moves, about var_tiles per CTA
            nC = (int)std::min<uint64_t>((uint64_t)c->cap_small,
                                         std::max<uint64_t>(1, cdiv(cdiv((uint64_t)sp->host.max_step_moves, 32),
                                                                    (uint64_t)c->var_tiles)));
            E.dyn_sync = !one_step && nC > 1;
        }
        // one CTA on one GPU, several steps, moves cached: the WORK rows live in the CTA's
        // shared memory (the kernel resolves WORK pointers there)
        const uint64_t wbytes = (uint64_t)dp.host.work_units * unit * (uint64_t)c->Rg;
        if (c->swork && !E.small_var && !E.small_own && nC <= 1 && c->G == 1 && !c->emulated && c->nprocs == 1 &&
            dp.nsteps > 1 && E.small_cache > 0 && c->p <= kRankTable && wbytes > 0 &&
            wbytes <= (uint64_t)kSmallWorkSmem)
            E.small_swork = 1;
        // few pieces per CTA and step: the smallest block (from small_nt = 64 threads) with one
        // piece per thread -- fewer idle warps contend for issue slots at every step (measured:
        // 4-5 % at <= 64 B; four pieces per thread in a smaller block lose up to 30 %)
        if (!E.small_var) {
            const uint64_t per_cta = cdiv(items, (uint64_t)std::max(1, nC));
            uint64_t nt = (uint64_t)c->small_nt;
            while (nt < 512 && (nt < per_cta || nt < (uint64_t)c->p || nt < (uint64_t)dp.nsteps)) nt *= 2;
            if (nt < 512) E.small_threads = (int32_t)nt;
        }
        // one step on one GPU, every move cached: the tiny kernel (no flags,
        // steps or rank tables -- the shortest instruction stream for a cold SM)
        tiny = c->tiny && one_step && c->G == 1 && !c->emulated && c->nprocs == 1 && !E.small_var &&
               !E.small_own && !E.small_ll && E.small_cache > 0 && sp == &dp;
        // several steps, one CTA, one GPU, every move cached: the tiny multi-step kernel
        const bool tiny_ms = c->tiny && !one_step && c->G == 1 && !c->emulated && c->nprocs == 1 &&
                             (nC <= 1 || E.small_own > 1) && !E.small_var && !E.dyn_sync && !E.small_ll &&
                             E.small_cache > 0 && dp.nsteps <= kMaxStepsSmem && sp == &dp;
        // one-step eager launches across GPUs: the tiny eager kernel (same word protocol)
        const bool tiny_ll = c->tiny && one_step && E.small_ll && !E.small_var && !E.small_own && E.small_cache > 0;
        if (tiny && c->tiny_even) {
            // the tiny kernel hands each CTA blockDim consecutive pieces: size the block to the
            // pieces the kernel decodes (fan-out: one per source piece, not per destination) over
            // the grid, a multiple of a warp, so every CTA of the grid gets work (measured, p = 8:
            // allgather 16 / 32 / 64 / 128 KiB 2.12 / 2.12 / 2.22 / 2.78 -> 1.50 / 1.55 / 1.59 /
            // 2.27 us -- the power-of-two block sized by fan-out-weighted pieces left 7 of 8 CTAs
            // idle; alltoall 16 KiB 1.52 -> 1.48)
            const uint64_t kitems = (uint64_t)dp.host.max_step_moves * ppm;
            const uint64_t nt = std::max<uint64_t>(64, std::min<uint64_t>(512, (cdiv(kitems, (uint64_t)std::max(1, nC)) + 31) / 32 * 32));
            E.small_threads = (int32_t)nt;
        }
        if (tiny) e = launch_tiny(E, std::max(1, nC), pdl && c->pdl, stream);
        else if (tiny_ms) {
            E.small_swork = 0;   // (the tiny multi-step kernel keeps WORK in global memory / L2)
            E.tiny_step_items = (int32_t)std::min<uint64_t>(INT32_MAX, (uint64_t)dp.host.max_step_moves * ppm);
            e = launch_tiny_ms(E, std::max(1, nC), pdl && c->pdl, stream);
        }
        else if (tiny_ll) {
            if (c->tiny_even) {   // (the same sizing: the pieces of the busiest GPU's eager program)
                const uint64_t kitems = (uint64_t)nmoves_g * ppm;
                E.small_threads = (int32_t)std::max<uint64_t>(
                    64, std::min<uint64_t>(512, (cdiv(kitems, (uint64_t)std::max(1, nC)) + 31) / 32 * 32));
            }
            coop = coop_level(c, !one_step && nC > 1 && !E.small_own);
            e = launch_tiny_ll(E, std::max(1, nC), c->emulated ? c->G : 1, coop, pdl && c->pdl, stream);
        } else {
            coop = coop_level(c, !one_step && nC > 1 && !E.small_own);
            e = launch_small(E, std::max(1, nC), c->emulated ? c->G : 1, coop, pdl && c->pdl, stream);
        }
        tiny = tiny || tiny_ll || tiny_ms;
    } else {
        int nC = gr.n();
        // dynamic mode: one step whose moves all fit the CTA's shared-memory move tile and
        // whose busiest GPU moves enough bytes for the tail of static slices to matter
        const int64_t ntiles = (dp.max_gpu_moves + kMoveTile - 1) / kMoveTile;
        if (c->dyn && dp.nsteps == 1 && ntiles <= kMaxDynTiles && dp.max_gpu_bytes_units > 0) {
            const uint64_t total = (uint64_t)dp.max_gpu_bytes_units * unit;
            const uint64_t avg = total / (uint64_t)std::max<int64_t>(1, dp.max_gpu_moves);
            // measured (p = 8..32 on one B200): the queues win once moves are large; with many
            // mid-size moves the per-tile setup costs more than the tail it removes
            if ((total >= c->dyn_min_total && avg >= kDynMinAvg) || (total >= kDynBigTotal && avg >= kDynMinMove)) {
                // the mid TMA ring at 2 CTAs / SM: twice the producers and LSU warps of the
                // big ring (the LSU queue needs the warps; the TMA queue is indifferent).  The
                // grid depends on the program only, so processes pair CTA flag slots 1:1.
                const TmaConfig tm = c->force_big > 0 ? kTmaBig : kTmaMid;
                E.stages = tm.stages;
                E.chunk = tm.chunk;
                E.ahead = tm.ahead;
                nC = c->force_big > 0 ? c->cap_big : c->cap_ctas;
                uint64_t U = total / ((uint64_t)nC * (uint64_t)c->dyn_pieces);
                U = std::max<uint64_t>((uint64_t)E.chunk, std::min<uint64_t>(U, kDynMaxPiece));
                // many move tiles (p >= 23 ranks on one GPU): each tile is classified by the whole
                // CTA while the producer stops issuing, so fewer, longer pieces pay (measured,
                // p = 32, 256 KiB blocks: 16 -> 48 KiB pieces, 93.2 -> 85.7 us; one or two
                // tiles: unchanged or slower)
                if (ntiles >= 4) U = std::max<uint64_t>(U, 3 * (uint64_t)E.chunk);
                U = U / (uint64_t)E.chunk * (uint64_t)E.chunk;
                E.nS = nC;
                E.nF = 1;
                E.dyn_units = (int32_t)std::max<int64_t>(1, ntiles);
                E.dyn_u = (int32_t)U;
            }
        } else if (c->dyn && dp.nsteps > 1 && dp.dyn_tiles <= kMaxDynTiles &&
                   (c->force_sync > 0 || (dp.host.max_step_moves >= kDynSyncMoves && (uint64_t)dp.host.max_step_units * unit >= kDynSyncMin) ||
                    // moves of different lengths: static flow groups get unequal byte counts
                    (!dp.uniform_len && (uint64_t)dp.host.max_step_units * unit >= kDynSyncMinUneven)) &&
                   c->force_sync != 0) {
            // multi-step dynamic mode: queues per step, a CTA barrier per GPU row between steps,
            // one flag per peer GPU (the flow-ownership rule no longer applies)
            const TmaConfig tm = c->force_big > 0 ? kTmaBig : kTmaMid;
            E.stages = tm.stages;
            E.chunk = tm.chunk;
            E.ahead = tm.ahead;
            nC = c->force_big > 0 ? c->cap_big : c->cap_ctas;
            const uint64_t total = (uint64_t)dp.host.max_step_units * unit;
            uint64_t U = total / ((uint64_t)nC * (uint64_t)c->dyn_pieces);
            U = std::max<uint64_t>((uint64_t)E.chunk, std::min<uint64_t>(U, kDynMaxPiece));
            U = U / (uint64_t)E.chunk * (uint64_t)E.chunk;
            E.nS = nC;
            E.nF = 1;
            E.dyn_units = (int32_t)dp.dyn_tiles;
            E.dyn_u = (int32_t)U;
            E.dyn_sync = 1;
        }
        // several GPUs: CTAs of a GPU meet at a GPU-scope counter barrier after each step and ONE
        // system-scope release per peer GPU signals it, instead of one per (CTA, peer): 296 CTAs
        // x (G-1) peers of microsecond releases per step otherwise (measured, 8 emulated GPUs:
        // ring allgather 16 KiB 341 -> 285 us, Bruck allgather 64 KiB 125 -> 102 us; single-step
        // launches unchanged)
        if (c->G > 1 && c->row_signal) {
            // (and the CTAs split the GPU's own moves evenly: the kernel's flow-group ranges
            // become move-index ranges, so step 0's flow-range prefetch does not apply)
            if (!E.dyn_units) E.d0_base = -1;
            E.dyn_sync = 1;
        }
        // warp-ring dynamic mode: when some moves may not be 16-B congruent, every warp streams
        // its own pieces through a TMA ring -- congruent ones with bulk stores, the others with
        // 16-B stores the warp shifts out of shared memory (exec_kernel.cu dyn_tile_w; measured,
        // cfg4 mean 4 MiB int64: 96.9 / 103.1 / 106.6 -> 92.3 / 87.2 / 100.6 us, seeds 0-2)
        // (measured, cfg4 int64, first version: the LSU path won below ~100 MiB per GPU -- mean
        // 1 MiB 24.3 vs 25.7 us -- and the warp rings above: mean 2 MiB 55.5 -> 51.9, 4 MiB 96.9
        // -> 92.3; with constant-shift stores the rings win from 1 MiB: kWringMinVol)
        const uint64_t wr_vol = dp.nsteps == 1 ? src_vol : step_vol;
        if (E.dyn_units && c->wring &&
            (c->wring == 2 ||
             (wr_vol >= kWringMinVol &&
              (unit % 16 || ((uintptr_t)send | (uintptr_t)recv | send_stride | recv_stride | E.work_stride) % 16)))) {
            E.wring = 1;
            E.wslack = c->wslack;
            E.chunk = kWChunk;
            E.stages = kWarpsExec * kWStages;   // dynamic smem = stages x chunk (every warp's ring)
            E.ahead = 0;
        }
        coop = coop_level(c, dp.nsteps > 1 && nC > 1);
        e = launch_exec(E, nC, c->emulated ? c->G : 1, coop, pdl && c->pdl, stream);
    }
    if (e != cudaSuccess) {
        if (getenv("MPXA_DEBUG")) fprintf(stderr, "mpxa: launch failed: %s\n", cudaGetErrorString(e));
        return MPXA_ERR_CUDA;
    }
    c->launches++;
    // execution path of this launch (tests assert the intended path ran: mpxa__last_launch)
    c->last_path = (small ? 1u : 0u) | (E.small_ll ? 2u : 0u) | (E.small_var ? 4u : 0u) |
                   (E.dyn_units ? 8u : 0u) | (E.dyn_sync ? 16u : 0u) | (E.small_own ? 32u : 0u) |
                   (E.small_swork ? 64u : 0u) | (E.wring ? 128u : 0u) | (tiny ? 256u : 0u) |
                   (coop ? 512u : 0u);
    return MPXA_SUCCESS;
}

// per-call program upload through a ring of pinned slots (stream-ordered, no host sync
// unless the ring wraps onto a copy still in flight)
int run_dynamic(mpxa_comm_t c, const Program &P, const char *send, char *recv, uint64_t unit,
                uint64_t send_stride, uint64_t recv_stride, cudaStream_t stream) {
    if (c->ring.empty()) c->ring.resize(8);
    Slot &s = c->ring[c->ring_next];
    c->ring_next = (c->ring_next + 1) % (int)c->ring.size();
    if (!s.ev) CK(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
    if (s.used) CK(cudaEventSynchronize(s.ev));
    size_t n = serialized_size(P);
    if (n > s.cap) {
        if (s.dmem) CK(cudaFree(s.dmem));
        CK(cudaMalloc(&s.dmem, n));
        s.cap = n;
    }
    if (n > s.pcap) {
        if (s.pinned) CK(cudaFreeHost(s.pinned));
        CK(cudaHostAlloc((void **)&s.pinned, n, cudaHostAllocDefault));
        s.pcap = n;
    }
    std::vector<char> buf;
    serialize(P, buf, (uintptr_t)s.dmem);
    memcpy(s.pinned, buf.data(), n);
    CK(cudaMemcpyAsync(s.dmem, s.pinned, n, cudaMemcpyHostToDevice, stream));
    DevProg dp;
    dp.per_call = true;
    dp.dmem = s.dmem;
    dp.gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + P.G);
    dp.bytes = n;
    dp.host = P;
    dp.nsteps = P.nsteps();
    prog_facts(dp);
    int rc = run_program(c, dp, send, recv, unit, send_stride, recv_stride, stream, nullptr, /*pdl=*/false);
    CK(cudaEventRecord(s.ev, stream));
    s.used = true;
    dp.dmem = nullptr;
    return rc;
}

// ---- argument checks (all before any data moves) -------------------------
bool overlap(const void *a, size_t na, const void *b, size_t nb) {
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return na && nb && x < y + nb && y < x + na;
}

int check_uniform(mpxa_comm_t c, const void *send, size_t count, size_t w, void *recv, int op) {
    if (!c) return MPXA_ERR_ARG;
    if (!dtype_ok(w)) return MPXA_ERR_ARG;
    if (count && (!send || !recv)) return MPXA_ERR_ARG;
    size_t blk = count * w;
    size_t sbytes = (op == MPXA_OP_ALLTOALL ? (size_t)c->p : 1) * blk * c->R;
    size_t rbytes = (size_t)c->p * blk * c->R;
    if (overlap(send, sbytes, recv, rbytes)) return MPXA_ERR_ARG;
    return MPXA_SUCCESS;
}

// Gather the FULL count/displacement matrices a v-schedule needs.  Single process: the
// caller's R*p rows are all p rows.  Multi-process: all-gather through the bootstrap
// (host collective; persistent requests pay it once at init).
// counts / displacements may live in device memory (SURVEY.md §8(b) ownership): such arrays
// are copied to the host first (a synchronous copy -- the persistent forms pay it once)
// Device-resident arrays of a one-shot call are read in the caller's stream order (async copy
// on `stream`, then a sync of that stream); at *_init (no stream) they must already be
// complete (the caller synchronized their producer), and a plain cudaMemcpy reads them.
int host_view(const int64_t *&a, size_t n, std::vector<int64_t> &store, cudaStream_t stream) {
    // recently seen HOST arrays skip the driver query (~1 us each): a host address never
    // becomes a device address (the driver's device VA range is reserved apart from the heap)
    static thread_local const void *known_host[8] = {};
    static thread_local int known_next = 0;
    for (const void *k : known_host)
        if (k == (const void *)a) return MPXA_SUCCESS;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, a) != cudaSuccess) {
        cudaGetLastError();   // unregistered host memory on older drivers: treat as host
        known_host[known_next] = a;
        known_next = (known_next + 1) & 7;
        return MPXA_SUCCESS;
    }
    if (at.type != cudaMemoryTypeDevice) {
        known_host[known_next] = a;
        known_next = (known_next + 1) & 7;
    }
    if (at.type == cudaMemoryTypeDevice) {
        store.resize(n);
        if (stream) {
            CK(cudaMemcpyAsync(store.data(), a, n * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
        } else {
            CK(cudaMemcpy(store.data(), a, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
        }
        a = store.data();
    }
    return MPXA_SUCCESS;
}

int gather_v(mpxa_comm_t c, const int64_t *sc, const int64_t *sd, const int64_t *rc,
             const int64_t *rd, size_t w, size_t send_bpr, size_t recv_bpr,
             std::vector<int64_t> &C, std::vector<int64_t> &SD, std::vector<int64_t> &RD, cudaStream_t stream) {
    const int p = c->p, R = c->R;
    if (!sc || !sd || !rc || !rd) return MPXA_ERR_ARG;
    std::vector<int64_t> hs[4];
    const size_t nrows = (size_t)R * p;
    int hr = host_view(sc, nrows, hs[0], stream);
    if (!hr) hr = host_view(sd, nrows, hs[1], stream);
    if (!hr) hr = host_view(rc, nrows, hs[2], stream);
    if (!hr) hr = host_view(rd, nrows, hs[3], stream);
    if (hr) return hr;
    for (int t = 0; t < R; t++)
        for (int j = 0; j < p; j++) {
            size_t i = (size_t)t * p + j;
            if (sc[i] < 0 || sd[i] < 0 || rc[i] < 0 || rd[i] < 0) return MPXA_ERR_ARG;
            if ((uint64_t)(sc[i] + sd[i]) * w > send_bpr) return MPXA_ERR_ARG;
            if ((uint64_t)(rc[i] + rd[i]) * w > recv_bpr) return MPXA_ERR_ARG;
        }
    size_t rows = (size_t)R * p;
    std::vector<int64_t> mine(rows * 4);
    memcpy(mine.data(), sc, rows * 8);
    memcpy(mine.data() + rows, sd, rows * 8);
    memcpy(mine.data() + 2 * rows, rc, rows * 8);
    memcpy(mine.data() + 3 * rows, rd, rows * 8);
    std::vector<int64_t> all(rows * 4 * c->nprocs);
    int r = bootstrap(c, mine.data(), all.data(), rows * 4 * 8);
    if (r) return r;
    C.assign((size_t)p * p, 0);
    SD.assign((size_t)p * p, 0);
    RD.assign((size_t)p * p, 0);
    std::vector<int64_t> RC((size_t)p * p);
    for (int q = 0; q < c->nprocs; q++) {
        const int64_t *b = all.data() + (size_t)q * rows * 4;
        for (size_t i = 0; i < rows; i++) {
            size_t gi = (size_t)q * rows + i;   // global row-major index (rank q*R + t, j)
            C[gi] = b[i];
            SD[gi] = b[rows + i];
            RC[gi] = b[2 * rows + i];
            RD[gi] = b[3 * rows + i];
        }
    }
    for (int s = 0; s < p; s++)   // SPEC.md:208 global consistency
        for (int j = 0; j < p; j++)
            if (C[(size_t)s * p + j] != RC[(size_t)j * p + s]) return MPXA_ERR_MISMATCH;
    return MPXA_SUCCESS;
}

constexpr size_t kVCacheMax = 32;

uint64_t fnv(uint64_t h, const void *p, size_t n) {   // FNV-1a over 8-byte words
    const unsigned char *b = (const unsigned char *)p;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        memcpy(&w, b + i, 8);
        h = (h ^ w) * 1099511628211ull;
    }
    for (; i < n; i++) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

// cached one-shot v-program (built and uploaded on a miss; LRU eviction waits for the
// evicted program's last launch)
int vprogram(mpxa_comm_t c, int algo, const std::vector<int64_t> &C, const std::vector<int64_t> &SD,
             const std::vector<int64_t> &RD, mpxa_comm_s::VEntry *&out) {
    uint64_t h = fnv(1469598103934665603ull, &algo, sizeof algo);
    h = fnv(h, C.data(), C.size() * 8);
    h = fnv(h, SD.data(), SD.size() * 8);
    h = fnv(h, RD.data(), RD.size() * 8);
    auto &bucket = c->vcache[h];
    for (auto &e : bucket)
        if (e.algo == algo && e.C == C && e.SD == SD && e.RD == RD) {
            e.used = ++c->vcache_clock;
            out = &e;
            return MPXA_SUCCESS;
        }
    if (c->vcache_n >= kVCacheMax) {            // evict the least recently used entry
        uint64_t best = ~0ull, bh = 0;
        size_t bi = 0;
        for (auto &kv : c->vcache)
            for (size_t i = 0; i < kv.second.size(); i++)
                if (kv.second[i].used < best) { best = kv.second[i].used; bh = kv.first; bi = i; }
        auto &vb = c->vcache[bh];
        // the evicted program may still be in flight on any stream (launches record no event:
        // eviction is rare, a device-wide sync there is cheaper than an event per call)
        CK(cudaDeviceSynchronize());
        if (vb[bi].last) cudaEventDestroy(vb[bi].last);
        if (vb[bi].prog) cudaFree(vb[bi].prog->dmem);
        vb.erase(vb.begin() + (long)bi);
        if (vb.empty()) c->vcache.erase(bh);
        c->vcache_n--;
    }
    Program P;
    if (!build_alltoallv(P, algo, c->p, c->Rg, c->G, c->g, C.data(), SD.data(), RD.data(), c->hier_staged))
        return MPXA_ERR_ALGO;
    mpxa_comm_s::VEntry e;
    e.algo = algo;
    e.C = C; e.SD = SD; e.RD = RD;
    int r = upload_program(P, e.prog);
    if (r) return r;
    CK(cudaEventCreateWithFlags(&e.last, cudaEventDisableTiming));
    e.used = ++c->vcache_clock;
    auto &b2 = c->vcache[h];
    b2.push_back(std::move(e));
    c->vcache_n++;
    out = &b2.back();
    return MPXA_SUCCESS;
}

int alltoallv_impl(const void *sendbuf, const int64_t *sc, const int64_t *sd, size_t send_bpr,
                   void *recvbuf, const int64_t *rc, const int64_t *rd, size_t recv_bpr, size_t w,
                   int algo, mpxa_comm_t c, cudaStream_t stream, mpxa_request_t *req) {
    if (!c) return MPXA_ERR_ARG;
    if (!dtype_ok(w)) return MPXA_ERR_ARG;
    if (!sendbuf || !recvbuf) return MPXA_ERR_ARG;
    if (overlap(sendbuf, send_bpr * c->R, recvbuf, recv_bpr * c->R)) return MPXA_ERR_ARG;
    if (algo != A_DEFAULT && !algo_valid(MPXA_OP_ALLTOALLV, algo)) return MPXA_ERR_ALGO;
    if (algo == A_HIER && c->p % c->g) return MPXA_ERR_TOPOLOGY;
    std::vector<int64_t> C, SD, RD;
    int r = gather_v(c, sc, sd, rc, rd, w, send_bpr, recv_bpr, C, SD, RD, stream);
    if (r) return r;
    if (algo == A_DEFAULT) {
        // the selector's size for a v-collective is the mean pair segment of the GLOBAL count
        // matrix (the same on every process; a local size such as this rank's recv capacity
        // could pick different variants on different processes)
        int64_t tot = 0;
        for (int64_t x : C) tot += x;
        const uint64_t mean = ((uint64_t)tot * w + (uint64_t)c->p * c->p - 1) / ((uint64_t)c->p * c->p);
        algo = default_algo(c, MPXA_OP_ALLTOALLV, mean);
        if (!algo_valid(MPXA_OP_ALLTOALLV, algo)) return MPXA_ERR_ALGO;
        if (algo == A_HIER && c->p % c->g) return MPXA_ERR_TOPOLOGY;
    }
    if (!req) {                                  // one-shot: cached program, PDL launch
        mpxa_comm_s::VEntry *e = nullptr;
        r = vprogram(c, algo, C, SD, RD, e);
        if (r) return r;
        return run_program(c, *e->prog, (const char *)sendbuf, (char *)recvbuf, w, send_bpr, recv_bpr, stream);
    }
    Program P;
    if (!build_alltoallv(P, algo, c->p, c->Rg, c->G, c->g, C.data(), SD.data(), RD.data(), c->hier_staged))
        return MPXA_ERR_ALGO;
    if (req) {
        auto q = new mpxa_request_s();
        q->comm = c; q->op = MPXA_OP_ALLTOALLV; q->algo = algo;
        int rc2 = upload_program(P, q->prog);
        if (rc2) { delete q; return rc2; }
        q->send = (const char *)sendbuf; q->recv = (char *)recvbuf;
        q->unit = w; q->send_stride = send_bpr; q->recv_stride = recv_bpr;
        q->grid = choose_grid(c, P, w);
        if (c->nprocs > 1) {
            rc2 = mpxa_register(c, recvbuf, recv_bpr * c->R);
            if (rc2) { delete q; return rc2; }
        }
        rc2 = ensure_work(c, (size_t)P.work_units * w * c->Rg);
        if (rc2) { delete q; return rc2; }
        prebuild_companions(c, *q->prog, w);
        *req = q;
        return MPXA_SUCCESS;
    }
    return MPXA_SUCCESS;
}

int uniform_impl(int op, const void *sendbuf, size_t count, size_t w, void *recvbuf, int algo,
                 mpxa_comm_t c, cudaStream_t stream, mpxa_request_t *req, int stage = -1,
                 bool force_bruck = false) {
    int rc = check_uniform(c, sendbuf, count, w, recvbuf, op);
    if (rc) return rc;
    const uint64_t unit = (uint64_t)count * w;
    if (force_bruck) algo = A_BRUCK;
    if (algo == A_DEFAULT) algo = default_algo(c, op, unit);
    if (!algo_valid(op, algo)) return MPXA_ERR_ALGO;
    if (algo == A_HIER && c->p % c->g) return MPXA_ERR_TOPOLOGY;
    std::shared_ptr<DevProg> dp;
    rc = cached_uniform(c, op, algo, stage, dp);
    if (rc) return rc;
    uint64_t sstride = op == MPXA_OP_ALLTOALL ? (uint64_t)c->p * unit : unit;
    uint64_t rstride = (uint64_t)c->p * unit;
    if (req) {
        auto q = new mpxa_request_s();
        q->comm = c; q->op = op; q->algo = algo; q->prog = dp;
        q->send = (const char *)sendbuf; q->recv = (char *)recvbuf;
        q->unit = unit; q->send_stride = sstride; q->recv_stride = rstride;
        q->grid = choose_grid(c, dp->host, unit);
        if (c->nprocs > 1 && unit) {
            rc = mpxa_register(c, recvbuf, rstride * c->R);
            if (rc) { delete q; return rc; }
        }
        rc = ensure_work(c, (size_t)dp->host.work_units * unit * c->Rg);
        if (rc) { delete q; return rc; }
        if (unit) prebuild_companions(c, *dp, unit);
        *req = q;
        return MPXA_SUCCESS;
    }
    if (unit == 0) return MPXA_SUCCESS;   // nothing moves; every process takes this branch
    return run_program(c, *dp, (const char *)sendbuf, (char *)recvbuf, unit, sstride, rstride, stream);
}

// f1: persistent / one-shot neighbor alltoallv.  Local per-edge arrays of
// this process's ranks are all-gathered into the global graph, validated and compiled.
int neighbor_impl(bool locality, const void *sendbuf, const int64_t *sc, const int64_t *sd, size_t send_bpr,
                  void *recvbuf, const int64_t *rc, const int64_t *rd, size_t recv_bpr, size_t w,
                  const int64_t *sidx, const int64_t *ridx, mpxa_topo_t topo, cudaStream_t stream,
                  mpxa_request_t *req) {
    if (!topo || !topo->comm) return MPXA_ERR_ARG;
    mpxa_comm_t c = topo->comm;
    if (!dtype_ok(w)) return MPXA_ERR_ARG;
    if ((topo->nout && (!sc || !sd)) || (topo->nin && (!rc || !rd))) return MPXA_ERR_ARG;
    if (!sendbuf || !recvbuf) return MPXA_ERR_ARG;
    if (overlap(sendbuf, send_bpr * c->R, recvbuf, recv_bpr * c->R)) return MPXA_ERR_ARG;
    // local bounds ("counts/displs address in-bounds disjoint regions")
    int64_t nsel = 0, nrel = 0;
    for (int64_t e = 0; e < topo->nout; e++) {
        if (sc[e] < 0 || sd[e] < 0 || (uint64_t)(sc[e] + sd[e]) * w > send_bpr) return MPXA_ERR_ARG;
        nsel += sc[e];
    }
    for (int64_t e = 0; e < topo->nin; e++) {
        if (rc[e] < 0 || rd[e] < 0 || (uint64_t)(rc[e] + rd[e]) * w > recv_bpr) return MPXA_ERR_ARG;
        nrel += rc[e];
    }
    if (locality && ((nsel && !sidx) || (nrel && !ridx))) return MPXA_ERR_ARG;
    std::vector<int64_t> SC, SD, RC, RD, SI, RI;
    int r = allgather_concat(c, sc, (size_t)topo->nout, SC);
    if (!r) r = allgather_concat(c, sd, (size_t)topo->nout, SD);
    if (!r) r = allgather_concat(c, rc, (size_t)topo->nin, RC);
    if (!r) r = allgather_concat(c, rd, (size_t)topo->nin, RD);
    if (!r && locality) r = allgather_concat(c, sidx, (size_t)nsel, SI);
    if (!r && locality) r = allgather_concat(c, ridx, (size_t)nrel, RI);
    if (r) return r;
    if (SC.size() != topo->dst.size() || RC.size() != topo->src.size()) return MPXA_ERR_MISMATCH;
    Program P;
    r = build_neighbor(P, locality, c->p, c->Rg, c->G, c->g, topo->indeg.data(), topo->src.data(), RC.data(),
                       RD.data(), topo->outdeg.data(), topo->dst.data(), SC.data(), SD.data(),
                       locality ? SI.data() : nullptr, locality ? RI.data() : nullptr, c->hier_staged);
    if (r) return r;
    if (req) {
        auto q = new mpxa_request_s();
        q->comm = c; q->op = MPXA_OP_NEIGHBOR_ALLTOALLV; q->algo = locality ? A_LOCALITY : A_PAIRWISE;
        int rc2 = upload_program(P, q->prog);
        if (rc2) { delete q; return rc2; }
        q->send = (const char *)sendbuf; q->recv = (char *)recvbuf;
        q->unit = w; q->send_stride = send_bpr; q->recv_stride = recv_bpr;
        q->grid = choose_grid(c, P, w);
        if (c->nprocs > 1) {
            rc2 = mpxa_register(c, recvbuf, recv_bpr * c->R);
            if (rc2) { delete q; return rc2; }
        }
        rc2 = ensure_work(c, (size_t)P.work_units * w * c->Rg);
        if (rc2) { delete q; return rc2; }
        prebuild_companions(c, *q->prog, w);
        *req = q;
        return MPXA_SUCCESS;
    }
    return run_dynamic(c, P, (const char *)sendbuf, (char *)recvbuf, w, send_bpr, recv_bpr, stream);
}

cudaStream_t S(mpxa_stream_t s) { return (cudaStream_t)s; }

int load_selector_file(mpxa_comm_t c, const char *path);

// Tuning knobs, the selector table and forced variants, read once per comm.
void read_knobs(mpxa_comm_t c) {
    if (const char *e = getenv("MPXA_NS")) c->force_ns = atoi(e);
    if (const char *e = getenv("MPXA_NF")) c->force_nf = atoi(e);
    if (const char *e = getenv("MPXA_TMA_BIG")) c->force_big = atoi(e);
    if (const char *e = getenv("MPXA_NO_SMALL")) c->force_exec = atoi(e) != 0;
    if (const char *e = getenv("MPXA_NO_PDL")) c->pdl = atoi(e) == 0;
    if (const char *e = getenv("MPXA_NO_DYN")) c->dyn = atoi(e) == 0;
    if (const char *e = getenv("MPXA_NO_WRING")) c->wring = atoi(e) == 0 ? 1 : 0;
    if (const char *e = getenv("MPXA_WRING")) c->wring = atoi(e);
    if (const char *e = getenv("MPXA_DYN_PIECES")) c->dyn_pieces = std::max(1, atoi(e));
    if (const char *e = getenv("MPXA_NO_TINY")) c->tiny = atoi(e) == 0;
    if (const char *e = getenv("MPXA_TINY_EVEN")) c->tiny_even = atoi(e) != 0;
    if (const char *e = getenv("MPXA_WSLACK")) c->wslack = std::max(1, std::min(kWStages - 1, atoi(e)));
    if (const char *e = getenv("MPXA_DYN_MIN")) c->dyn_min_total = strtoull(e, nullptr, 10);
    if (const char *e = getenv("MPXA_DYN_SYNC")) c->force_sync = atoi(e);
    if (const char *e = getenv("MPXA_NO_SMALL_SYNC")) c->small_sync = atoi(e) == 0;
    if (const char *e = getenv("MPXA_SMALL_MAX")) c->small_max1 = strtoull(e, nullptr, 10);
    if (const char *e = getenv("MPXA_SMALL_VOL")) c->small_vol1 = strtoull(e, nullptr, 10);
    if (const char *e = getenv("MPXA_VAR_CHOP")) c->var_chop = atoll(e);
    if (const char *e = getenv("MPXA_VAR_TILES")) c->var_tiles = std::max(1, atoi(e));
    if (const char *e = getenv("MPXA_SWORK")) c->swork = atoi(e) != 0;
    if (const char *e = getenv("MPXA_SMALL_NT")) c->small_nt = std::max(32, std::min(512, atoi(e)));
    if (const char *e = getenv("MPXA_NO_LL")) c->ll = atoi(e) == 0;
    if (const char *e = getenv("MPXA_ONE_CTA_ITEMS")) c->one_cta_items = strtoull(e, nullptr, 10);
    if (const char *e = getenv("MPXA_OWN_VOL")) c->own_vol = strtoull(e, nullptr, 10);
    if (const char *e = getenv("MPXA_OWN_PER_CTA")) c->own_per_cta = strtoull(e, nullptr, 10);
    if (const char *e = getenv("MPXA_SMALL_ITEMS")) c->small_items = std::max<uint64_t>(64, strtoull(e, nullptr, 10));
    if (const char *e = getenv("MPXA_HIER_STAGED")) c->hier_staged = atoi(e) != 0;
    if (const char *e = getenv("MPXA_ROW_SIGNAL")) c->row_signal = atoi(e) != 0;
    if (const char *e = getenv("MPXA_LL_MAX")) c->ll_max = atoll(e);
    if (const char *e = getenv("MPXA_LL_MAX_MS")) c->ll_max_ms = atoll(e);
    // measured selector table: $MPXA_SELECTOR, else selector_b200.txt next to libmpxa.so
    // (an absent or unreadable file leaves the built-in rules)
    if (const char *sel = getenv("MPXA_SELECTOR")) {
        load_selector_file(c, sel);
    } else {
        Dl_info info;
        if (dladdr((void *)&read_knobs, &info) && info.dli_fname) {
            std::string path(info.dli_fname);
            auto slash = path.rfind('/');
            path = (slash == std::string::npos ? std::string(".") : path.substr(0, slash)) + "/selector_b200.txt";
            load_selector_file(c, path.c_str());
        }
    }
    if (const char *al = getenv("MPXA_ALGO")) {   // e.g. "alltoall:bruck,allgather:ring"
        std::stringstream ss{std::string(al)};
        std::string item;
        while (std::getline(ss, item, ',')) {
            auto k = item.find(':');
            if (k == std::string::npos) continue;
            std::string o = item.substr(0, k), v = item.substr(k + 1);
            int op = o == "alltoall" ? 0 : o == "alltoallv" ? 1 : o == "allgather" ? 2 : -1;
            int av = v == "pairwise" ? 1 : v == "bruck" ? 2 : v == "hier" ? 3 : v == "ring" ? 4 : 0;
            if (op >= 0 && algo_valid(op, av)) c->user_algo[op] = av;
        }
    }
}

// Digest of everything that chooses a launch's protocol, path or grid on the host: every
// knob, the selector table, the forced variants and the initial heap size (heap growth is
// a collective IPC exchange: the sizes must evolve identically on every process).
uint64_t knob_digest(mpxa_comm_t c, size_t heap) {
    const int64_t v[] = {c->force_ns, c->force_nf, c->force_big, c->force_exec, c->pdl, c->dyn, c->wring, c->wslack, c->tiny, c->tiny_even, c->dyn_pieces,
                         (int64_t)c->dyn_min_total, c->force_sync, c->small_sync, (int64_t)c->small_max1,
                         (int64_t)c->small_vol1, c->var_chop, c->var_tiles, c->swork, c->small_nt, c->ll,
                         (int64_t)c->one_cta_items, (int64_t)c->small_items, (int64_t)c->own_vol,
                         (int64_t)c->own_per_cta, c->hier_staged, c->row_signal, c->ll_max, c->ll_max_ms,
                         c->user_algo[0], c->user_algo[1], c->user_algo[2], (int64_t)heap,
                         (int64_t)c->selector.size()};
    uint64_t h = fnv(1469598103934665603ull, v, sizeof v);
    for (const SelEntry &e : c->selector) {
        const int64_t r[] = {e.op, e.p, e.R, e.G, e.g, (int64_t)e.max_bytes, e.algo};
        h = fnv(h, r, sizeof r);
    }
    return h;
}

}  // namespace

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

const char *mpxa_error_string(int s) {
    switch (s) {
        case MPXA_SUCCESS: return "success";
        case MPXA_ERR_ARG: return "invalid argument";
        case MPXA_ERR_ALGO: return "unknown or unsupported algorithm for this operation";
        case MPXA_ERR_LIFECYCLE: return "request lifecycle violation";
        case MPXA_ERR_TOPOLOGY: return "invalid rank / group topology";
        case MPXA_ERR_MISMATCH: return "argument mismatch across processes";
        case MPXA_ERR_CUDA: return "CUDA error";
        case MPXA_ERR_TIMEOUT: return "device watchdog timeout (communicator poisoned)";
        case MPXA_ERR_NOMEM: return "out of memory";
        case MPXA_ERR_UNREGISTERED: return "recvbuf not registered (multi-process mode)";
        default: return "unknown status";
    }
}

const char *mpxa_algo_name(mpxa_algo_t a) {
    switch (a) {
        case MPXA_ALGO_DEFAULT: return "default";
        case MPXA_ALGO_PAIRWISE: return "pairwise";
        case MPXA_ALGO_BRUCK: return "bruck";
        case MPXA_ALGO_HIER: return "hier";
        case MPXA_ALGO_RING: return "ring";
        case MPXA_ALGO_LOCALITY: return "locality";
        default: return "unknown";
    }
}

int mpxa_init(mpxa_comm_t *out, const mpxa_init_args *a) {
    if (!out || !a) return MPXA_ERR_ARG;
    *out = nullptr;
    if (a->nprocs < 1 || a->proc < 0 || a->proc >= a->nprocs || a->ranks_per_proc < 1) return MPXA_ERR_TOPOLOGY;
    if (a->nprocs > 1 && !a->bootstrap_allgather) return MPXA_ERR_ARG;
    if (a->nprocs > 1 && a->emulate_gpus > 1) return MPXA_ERR_ARG;
    std::unique_ptr<mpxa_comm_s> c(new mpxa_comm_s());
    c->nprocs = a->nprocs;
    c->proc = a->proc;
    c->R = a->ranks_per_proc;
    c->device = a->device;
    c->p = c->nprocs * c->R;

    c->boot = a->bootstrap_allgather;
    c->ctx = a->ctx;
    c->timeout_s = a->timeout_s > 0 ? a->timeout_s : 60.0;
    if (a->emulate_gpus > 1) {
        if (c->R % a->emulate_gpus) return MPXA_ERR_TOPOLOGY;
        c->emulated = true;
        c->G = a->emulate_gpus;
        c->Rg = c->R / c->G;
    } else {
        c->G = c->nprocs;
        c->Rg = c->R;
    }
    // default group: the ranks of one (possibly emulated) GPU (Q6)
    c->g = a->group_size > 0 ? a->group_size : c->Rg;
    if (c->p % c->g) return MPXA_ERR_TOPOLOGY;
    if (c->G > kMaxGpus || c->p > 65535) return MPXA_ERR_TOPOLOGY;
    read_knobs(c.get());
    size_t heap = a->heap_bytes ? a->heap_bytes : (size_t)64 << 20;
    c->heap0 = heap;
    if (c->nprocs > 1) {
        // Every process must run the same protocol: the topology, every effective tuning knob,
        // the selector table and the forced variants are compared BEFORE any CUDA call (all
        // processes see all digests, so all return the same verdict -- no one is left waiting
        // in a later collective step).  A difference is MPXA_ERR_MISMATCH.
        uint64_t mine[5] = {(uint64_t)c->R, (uint64_t)c->g, (uint64_t)c->nprocs, knob_digest(c.get(), heap),
                            (uint64_t)(a->emulate_gpus > 1 ? a->emulate_gpus : 0)};
        std::vector<uint64_t> all(5 * (size_t)c->nprocs);
        int rc = bootstrap(c.get(), mine, all.data(), sizeof mine);
        if (rc) return rc;
        for (int q = 0; q < c->nprocs; q++)
            if (memcmp(mine, &all[5 * (size_t)q], sizeof mine)) return MPXA_ERR_MISMATCH;
    }
    CK(cudaSetDevice(c->device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, c->device));
    c->sm_count = prop.multiProcessorCount;
    int occ = std::max(1, exec_max_ctas_per_sm((size_t)kTmaMid.stages * kTmaMid.chunk));
    int occ_big = std::max(1, exec_max_ctas_per_sm((size_t)kTmaBig.stages * kTmaBig.chunk));
    int cap = std::min(kMaxCtas, c->sm_count * occ);
    int capb = std::min(kMaxCtas, c->sm_count * occ_big);
    if (c->emulated) { cap = std::max(1, cap / c->G); capb = std::max(1, capb / c->G); }
    c->cap_ctas = cap;
    c->cap_big = capb;
    c->cap_small = std::max(1, (c->emulated ? c->sm_count / c->G : c->sm_count));
    if (getenv("MPXA_DEBUG"))
        fprintf(stderr, "mpxa: %d SMs, executor CTAs/SM mid %d big %d -> caps %d / %d\n", c->sm_count, occ, occ_big,
                c->cap_ctas, c->cap_big);
    CK(cudaHostAlloc((void **)&c->err_host, sizeof(int32_t), cudaHostAllocMapped));
    *c->err_host = 0;
    CK(cudaHostGetDevicePointer((void **)&c->err_dev, c->err_host, 0));
    int nsym = c->emulated ? c->G : 1;
    CK(cudaMalloc((void **)&c->sym_local, sizeof(SymRegion) * nsym));
    CK(cudaMemset(c->sym_local, 0, sizeof(SymRegion) * nsym));
    CK(cudaMalloc((void **)&c->dc, sizeof(DevComm)));
    CK(cudaMemset(c->dc, 0, sizeof(DevComm)));
    memset(&c->dc_host, 0, sizeof(DevComm));
    if (c->nprocs > 1) {
        // the grid of a launch is computed from the CTA caps, and processes pair CTA flag
        // slots 1:1 -- the devices must agree on them (SM count, occupancy)
        uint64_t mine[3] = {(uint64_t)c->cap_ctas, (uint64_t)c->cap_big, (uint64_t)c->cap_small};
        std::vector<uint64_t> all(3 * (size_t)c->nprocs);
        int rc = bootstrap(c.get(), mine, all.data(), sizeof mine);
        if (rc) return rc;
        for (int q = 0; q < c->nprocs; q++)
            if (memcmp(mine, &all[3 * (size_t)q], sizeof mine)) return MPXA_ERR_MISMATCH;
        rc = ipc_exchange(c.get(), c->sym_local, (char **)c->sym_map);
        if (rc) return rc;
    } else {
        for (int g = 0; g < c->G; g++) c->sym_map[g] = c->sym_local + g;
    }
    int rc = ensure_work(c.get(), heap);
    if (rc) return rc;
    CK(cudaDeviceSynchronize());
    *out = c.release();
    return MPXA_SUCCESS;
}

int mpxa_finalize(mpxa_comm_t c) {
    if (!c) return MPXA_ERR_ARG;
    cudaDeviceSynchronize();
    if (c->nprocs > 1) {
        for (int d = 0; d < c->nprocs; d++) {
            if (d == c->proc) continue;
            if (c->sym_map[d]) cudaIpcCloseMemHandle(c->sym_map[d]);
            if (c->work_map[d]) cudaIpcCloseMemHandle(c->work_map[d]);
            for (auto &w : c->win_map)
                if (w.size() > (size_t)d && w[d]) cudaIpcCloseMemHandle(w[d]);
        }
    }
    for (auto &kv : c->ipc_opened) cudaIpcCloseMemHandle(kv.second);
    if (c->nprocs > 1)
        for (int d = 0; d < (int)c->part_map.size(); d++)
            if (d != c->proc && c->part_map[d]) cudaIpcCloseMemHandle(c->part_map[d]);
    if (c->part_local) cudaFree(c->part_local);
    if (c->pquery) cudaStreamDestroy(c->pquery);
    for (auto &kv : c->cache) cudaFree(kv.second->dmem);
    for (auto &kv : c->vcache)
        for (auto &e : kv.second) {
            if (e.prog) cudaFree(e.prog->dmem);
            if (e.last) cudaEventDestroy(e.last);
        }
    for (auto &s : c->ring) {
        if (s.dmem) cudaFree(s.dmem);
        if (s.pinned) cudaFreeHost(s.pinned);
        if (s.ev) cudaEventDestroy(s.ev);
    }
    if (c->work_local) cudaFree(c->work_local);
    if (c->sym_local) cudaFree(c->sym_local);
    if (c->dc) cudaFree(c->dc);
    if (c->err_host) cudaFreeHost(c->err_host);
    if (c->counts_tmp) cudaFree(c->counts_tmp);
    delete c;
    return MPXA_SUCCESS;
}

int mpxa_comm_size(mpxa_comm_t c, int *p) {
    if (!c || !p) return MPXA_ERR_ARG;
    *p = c->p;
    return MPXA_SUCCESS;
}

int mpxa_comm_rank0(mpxa_comm_t c, int *r0) {
    if (!c || !r0) return MPXA_ERR_ARG;
    *r0 = c->proc * c->R;
    return MPXA_SUCCESS;
}

int mpxa_comm_check(mpxa_comm_t c) {
    if (!c) return MPXA_ERR_ARG;
    if (c->err_host && *(volatile int32_t *)c->err_host) c->poisoned = true;
    return c->poisoned ? MPXA_ERR_TIMEOUT : MPXA_SUCCESS;
}

int mpxa_launch_count(mpxa_comm_t c, uint64_t *n) {
    if (!c || !n) return MPXA_ERR_ARG;
    *n = c->launches;
    return MPXA_SUCCESS;
}

int mpxa_register(mpxa_comm_t c, void *ptr, size_t bytes) {
    if (!c || !ptr) return MPXA_ERR_ARG;
    if (c->nprocs == 1) return MPXA_SUCCESS;
    uintptr_t x = (uintptr_t)ptr;
    // already inside a registered window?  (collective decision: every process registers
    // a buffer of its own, so all take the same branch only if all hit -- exchange a flag)
    int hit = 0;
    for (auto &w : c->windows)
        if (x >= w.base && x + bytes <= w.base + w.size) hit = 1;
    std::vector<int> hits(c->nprocs);
    int rc = bootstrap(c, &hit, hits.data(), sizeof hit);
    if (rc) return rc;
    bool all = true;
    for (int h : hits) all = all && h;
    if (all) return MPXA_SUCCESS;
    if (c->windows.size() >= (size_t)kMaxWindows) return MPXA_ERR_NOMEM;
    // allocation range of ptr: resolve through the driver entry point (no libcuda link)
    typedef int (*range_fn)(uintptr_t *, size_t *, uintptr_t);
    static range_fn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
        fn = (range_fn)f;
    }
    uintptr_t base = 0;
    size_t size = 0;
    if (!fn || fn(&base, &size, x) != 0) return MPXA_ERR_ARG;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, (void *)base));
    std::vector<cudaIpcMemHandle_t> allh(c->nprocs);
    rc = bootstrap(c, &h, allh.data(), sizeof h);
    if (rc) return rc;
    std::vector<char *> mapped(c->nprocs, nullptr);
    for (int d = 0; d < c->nprocs; d++) {
        if (d == c->proc) { mapped[d] = (char *)base; continue; }
        void *m = nullptr;
        CK(cudaIpcOpenMemHandle(&m, allh[d], cudaIpcMemLazyEnablePeerAccess));
        mapped[d] = (char *)m;
    }
    int wi = (int)c->windows.size();
    c->windows.push_back(Window{base, size});
    c->win_map.push_back(mapped);
    for (int d = 0; d < c->nprocs; d++) c->dc_host.win_table[(size_t)d * kMaxWindows + wi] = mapped[d];
    CK(cudaDeviceSynchronize());
    return upload_tables(c);
}

int mpxa_deregister(mpxa_comm_t c, void *ptr) {
    if (!c || !ptr) return MPXA_ERR_ARG;
    return MPXA_SUCCESS;   // windows live until finalize (indices must stay stable)
}

int mpxa_alltoall(const void *s, size_t count, size_t w, void *r, mpxa_comm_t c, mpxa_stream_t st) {
    return uniform_impl(MPXA_OP_ALLTOALL, s, count, w, r, A_DEFAULT, c, S(st), nullptr);
}
int mpxa_allgather(const void *s, size_t count, size_t w, void *r, mpxa_comm_t c, mpxa_stream_t st) {
    return uniform_impl(MPXA_OP_ALLGATHER, s, count, w, r, A_DEFAULT, c, S(st), nullptr);
}
int mpxa_alltoall_algo(const void *s, size_t count, size_t w, void *r, mpxa_algo_t a, mpxa_comm_t c,
                       mpxa_stream_t st) {
    return uniform_impl(MPXA_OP_ALLTOALL, s, count, w, r, a, c, S(st), nullptr);
}
int mpxa_allgather_algo(const void *s, size_t count, size_t w, void *r, mpxa_algo_t a, mpxa_comm_t c,
                        mpxa_stream_t st) {
    return uniform_impl(MPXA_OP_ALLGATHER, s, count, w, r, a, c, S(st), nullptr);
}
int mpxa_alltoallv(const void *s, const int64_t *sc, const int64_t *sd, size_t sb, void *r,
                   const int64_t *rc, const int64_t *rd, size_t rb, size_t w, mpxa_comm_t c,
                   mpxa_stream_t st) {
    return alltoallv_impl(s, sc, sd, sb, r, rc, rd, rb, w, A_DEFAULT, c, S(st), nullptr);
}
int mpxa_alltoallv_algo(const void *s, const int64_t *sc, const int64_t *sd, size_t sb, void *r,
                        const int64_t *rc, const int64_t *rd, size_t rb, size_t w, mpxa_algo_t a,
                        mpxa_comm_t c, mpxa_stream_t st) {
    return alltoallv_impl(s, sc, sd, sb, r, rc, rd, rb, w, a, c, S(st), nullptr);
}

int mpxa_alltoall_bruck_stage(const void *s, size_t count, size_t w, void *T, int stage, mpxa_comm_t c,
                              mpxa_stream_t st) {
    if (!c) return MPXA_ERR_ARG;
    if (stage < -1 || stage > ceil_log2(c->p)) return MPXA_ERR_ARG;
    return uniform_impl(MPXA_OP_ALLTOALL, s, count, w, T, A_BRUCK, c, S(st), nullptr, stage, true);
}
int mpxa_allgather_bruck_stage(const void *s, size_t count, size_t w, void *T, int stage, mpxa_comm_t c,
                               mpxa_stream_t st) {
    if (!c) return MPXA_ERR_ARG;
    if (stage < -1 || stage > ceil_log2(c->p)) return MPXA_ERR_ARG;
    return uniform_impl(MPXA_OP_ALLGATHER, s, count, w, T, A_BRUCK, c, S(st), nullptr, stage, true);
}

int mpxa_alltoallv_counts(const int64_t *d_sc, int64_t *d_rc, int64_t *d_rd, mpxa_comm_t c,
                          mpxa_stream_t st) {
    if (!c || !d_sc || !d_rc || !d_rd) return MPXA_ERR_ARG;
    if (c->poisoned) return MPXA_ERR_TIMEOUT;
    if (c->nprocs == 1 && !c->emulated) {
        // all p ranks are on this device: one kernel, transpose + warp scans
        cudaError_t e = launch_counts(d_sc, d_rc, d_rd, c->p, 0, c->p, S(st));
        if (e != cudaSuccess) return MPXA_ERR_CUDA;
        c->launches++;
        return MPXA_SUCCESS;
    }
    // multi-process (and emulated GPUs, which run the same protocol): an alltoall of one
    // int64 per rank pair into registered staging, then the scan kernel (2 launches)
    size_t bytes = (size_t)c->R * c->p * sizeof(int64_t);
    if (!c->counts_tmp) {
        CK(cudaMalloc((void **)&c->counts_tmp, bytes));
        c->counts_tmp_bytes = bytes;
        int rc = mpxa_register(c, c->counts_tmp, bytes);
        if (rc) return rc;
    }
    int rc = uniform_impl(MPXA_OP_ALLTOALL, d_sc, 1, 8, c->counts_tmp, A_PAIRWISE, c, S(st), nullptr);
    if (rc) return rc;
    cudaError_t e = launch_scan(c->counts_tmp, d_rc, d_rd, c->p, c->R, S(st));
    if (e != cudaSuccess) return MPXA_ERR_CUDA;
    c->launches++;
    return MPXA_SUCCESS;
}

// ---- persistent requests ----------------------------------------------------------------
int mpxa_alltoall_init(const void *s, size_t count, size_t w, void *r, mpxa_algo_t a, mpxa_comm_t c,
                       const void *info, mpxa_request_t *req) {
    (void)info;
    if (!req) return MPXA_ERR_ARG;
    *req = nullptr;
    return uniform_impl(MPXA_OP_ALLTOALL, s, count, w, r, a, c, nullptr, req);
}
int mpxa_allgather_init(const void *s, size_t count, size_t w, void *r, mpxa_algo_t a, mpxa_comm_t c,
                        const void *info, mpxa_request_t *req) {
    (void)info;
    if (!req) return MPXA_ERR_ARG;
    *req = nullptr;
    return uniform_impl(MPXA_OP_ALLGATHER, s, count, w, r, a, c, nullptr, req);
}
int mpxa_alltoallv_init(const void *s, const int64_t *sc, const int64_t *sd, size_t sb, void *r,
                        const int64_t *rc, const int64_t *rd, size_t rb, size_t w, mpxa_algo_t a,
                        mpxa_comm_t c, const void *info, mpxa_request_t *req) {
    (void)info;
    if (!req) return MPXA_ERR_ARG;
    *req = nullptr;
    return alltoallv_impl(s, sc, sd, sb, r, rc, rd, rb, w, a, c, nullptr, req);
}

int mpxa_start(mpxa_request_t q, mpxa_stream_t st) {
    if (!q) return MPXA_ERR_ARG;
    if (q->active) return MPXA_ERR_LIFECYCLE;
    mpxa_comm_t c = q->comm;
    if (q->pkind) {                     // partitioned end: begin the next cycle
        if (!q->matched) return MPXA_ERR_LIFECYCLE;
        if (c->poisoned) return MPXA_ERR_TIMEOUT;
        cudaError_t e = launch_part_start(q->pkind == 1, q->mycycle, q->cts_remote, S(st));
        if (e != cudaSuccess) return MPXA_ERR_CUDA;
        c->launches++;
        q->cycle++;
        if (q->pkind == 1) std::fill(q->readied.begin(), q->readied.end(), 0);
        q->active = true;
        return MPXA_SUCCESS;
    }
    if (c->active && c->active != q) return MPXA_ERR_LIFECYCLE;   // one in flight
    if (q->unit) {
        int rc = run_program(c, *q->prog, q->send, q->recv, q->unit, q->send_stride, q->recv_stride, S(st), &q->grid);
        if (rc) return rc;
    }
    // (no event here: mpxa_wait on the start stream -- the common case -- needs none; a wait on
    // another stream records one on the start stream then, which also covers any work queued
    // there after the start: conservative, never too early)
    q->start_stream = S(st);
    q->active = true;
    c->active = q;
    return MPXA_SUCCESS;
}

int mpxa_wait(mpxa_request_t q, mpxa_stream_t st) {
    if (!q) return MPXA_ERR_ARG;
    if (!q->active) return MPXA_ERR_LIFECYCLE;
    if (q->pkind) {                     // every partition of the cycle delivered / arrived
        const unsigned long long *flags = q->pkind == 1 ? q->sdev.arr : q->arr;
        const int n = q->pkind == 1 ? q->nparts : q->peer_nparts;
        cudaError_t e = launch_part_wait(flags, 0, n, q->mycycle, q->comm->err_dev,
                                         (long long)(q->comm->timeout_s * 1e9), S(st));
        if (e != cudaSuccess) return MPXA_ERR_CUDA;
        q->comm->launches++;
        q->active = false;
        return MPXA_SUCCESS;
    }
    if (S(st) != q->start_stream) {
        if (!q->done) CK(cudaEventCreateWithFlags(&q->done, cudaEventDisableTiming));
        CK(cudaEventRecord(q->done, q->start_stream));
        CK(cudaStreamWaitEvent(S(st), q->done, 0));
    }
    q->active = false;
    if (q->comm->active == q) q->comm->active = nullptr;
    return MPXA_SUCCESS;
}

int mpxa_request_free(mpxa_request_t *qp) {
    if (!qp || !*qp) return MPXA_ERR_ARG;
    mpxa_request_t q = *qp;
    if (q->active) return MPXA_ERR_LIFECYCLE;
    if (q->pkind) {                     // unmatched ends leave the pending list
        auto &pp = q->comm->ppending;
        pp.erase(std::remove(pp.begin(), pp.end(), q), pp.end());
    }
    if (q->done) cudaEventDestroy(q->done);
    // cached uniform programs are shared with the comm; v-programs are owned
    if ((q->op == MPXA_OP_ALLTOALLV || q->op == MPXA_OP_NEIGHBOR_ALLTOALLV) && q->prog && q->prog.use_count() == 1) {
        cudaDeviceSynchronize();
        cudaFree(q->prog->dmem);
    }
    delete q;
    *qp = nullptr;
    return MPXA_SUCCESS;
}

int mpxa_request_algorithm(mpxa_request_t q, mpxa_algo_t *a) {
    if (!q || !a) return MPXA_ERR_ARG;
    *a = (mpxa_algo_t)q->algo;
    return MPXA_SUCCESS;
}

// ---- partitioned point-to-point ---------------------------------------
namespace {
constexpr uint64_t kPartHeapSlots = 1u << 17;   // 1 MiB of 8-byte slots per process

int part_init_common(mpxa_comm_t c, void *buf, int partitions, size_t count, size_t w, int rank, int peer, int tag,
                     int kind, mpxa_request_t *req) {
    if (!c || !req) return MPXA_ERR_ARG;
    *req = nullptr;
    if (partitions < 1 || !dtype_ok(w) || (count && !buf)) return MPXA_ERR_ARG;
    const int r0 = c->proc * c->R;
    if (rank < r0 || rank >= r0 + c->R || peer < 0 || peer >= c->p) return MPXA_ERR_ARG;
    auto q = new mpxa_request_s();
    q->comm = c;
    q->op = -1;
    q->pkind = kind;
    q->prank = rank;
    q->ppeer = peer;
    q->ptag = tag;
    q->nparts = partitions;
    q->part_bytes = (uint64_t)count * w;
    q->pbuf = (char *)buf;
    c->ppending.push_back(q);
    *req = q;
    return MPXA_SUCCESS;
}

// device pointer of slot `off` in process `proc`'s partition heap
unsigned long long *pslot(mpxa_comm_t c, int proc, uint64_t off) { return c->part_map[proc] + off; }
}  // namespace

int mpxa_psend_init(const void *buf, int partitions, size_t count, size_t w, int rank, int dest, int tag,
                    mpxa_comm_t c, const void *info, mpxa_request_t *req) {
    (void)info;
    return part_init_common(c, (void *)buf, partitions, count, w, rank, dest, tag, 1, req);
}

int mpxa_precv_init(void *buf, int partitions, size_t count, size_t w, int rank, int source, int tag,
                    mpxa_comm_t c, const void *info, mpxa_request_t *req) {
    (void)info;
    return part_init_common(c, buf, partitions, count, w, rank, source, tag, 2, req);
}

int mpxa_pmatch(mpxa_comm_t c) {
    if (!c) return MPXA_ERR_ARG;
    // partition heap (first match only): allocate, zero, map every process's heap
    if (!c->part_local) {
        CK(cudaMalloc((void **)&c->part_local, kPartHeapSlots * 8));
        CK(cudaMemset(c->part_local, 0, kPartHeapSlots * 8));
        c->part_map.assign(c->nprocs, nullptr);
        c->part_cursor.assign(c->nprocs, 0);
        if (c->nprocs > 1) {
            std::vector<char *> m(c->nprocs);
            int rc = ipc_exchange(c, c->part_local, m.data());
            if (rc) return rc;
            for (int q = 0; q < c->nprocs; q++) c->part_map[q] = (unsigned long long *)m[q];
        } else {
            c->part_map[0] = c->part_local;
        }
        CK(cudaStreamCreateWithFlags(&c->pquery, cudaStreamNonBlocking));
    }
    // every process's pending ends (creation order) with the IPC handle of recv buffers
    struct Rec {
        int32_t kind, rank, peer, tag, nparts, proc;
        uint64_t part_bytes, idx, buf_off;
        cudaIpcMemHandle_t h;
    };
    std::vector<Rec> mine;
    for (size_t i = 0; i < c->ppending.size(); i++) {
        mpxa_request_t q = c->ppending[i];
        Rec r{};
        r.kind = q->pkind; r.rank = q->prank; r.peer = q->ppeer; r.tag = q->ptag; r.nparts = q->nparts;
        r.proc = c->proc; r.part_bytes = q->part_bytes; r.idx = i;
        if (q->pkind == 2 && c->nprocs > 1 && q->part_bytes) {
            static int (*range_fn)(uintptr_t *, size_t *, uintptr_t) = nullptr;
            if (!range_fn) {
                void *f = nullptr;
                cudaDriverEntryPointQueryResult qr;
                CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &qr));
                range_fn = (int (*)(uintptr_t *, size_t *, uintptr_t))f;
            }
            uintptr_t base = 0;
            size_t size = 0;
            if (!range_fn || range_fn(&base, &size, (uintptr_t)q->pbuf) != 0) return MPXA_ERR_ARG;
            CK(cudaIpcGetMemHandle(&r.h, (void *)base));
            r.buf_off = (uintptr_t)q->pbuf - base;
        }
        mine.push_back(r);
    }
    std::vector<Rec> all;
    int rc = allgather_concat(c, mine.data(), mine.size(), all);
    if (rc) return rc;
    // pair: every send with the first unmatched receive of (dest <- rank, tag), global order
    std::vector<int> partner(all.size(), -1);
    for (size_t i = 0; i < all.size(); i++) {
        if (all[i].kind != 1) continue;
        for (size_t j = 0; j < all.size(); j++)
            if (all[j].kind == 2 && partner[j] < 0 && all[j].rank == all[i].peer && all[j].peer == all[i].rank &&
                all[j].tag == all[i].tag) {
                partner[i] = (int)j;
                partner[j] = (int)i;
                break;
            }
    }
    for (size_t i = 0; i < all.size(); i++) {
        if (partner[i] < 0) return MPXA_ERR_MISMATCH;
        const Rec &a = all[i], &b = all[partner[i]];
        if ((uint64_t)a.nparts * a.part_bytes != (uint64_t)b.nparts * b.part_bytes) return MPXA_ERR_MISMATCH;
    }
    // slots, identical on every process: receiver heap: rcycle, arr[n_s]; sender heap: scycle,
    // cts, done[n_s]
    for (size_t i = 0; i < all.size(); i++) {
        if (all[i].kind != 1) continue;
        const Rec &sd = all[i], &rv = all[partner[i]];
        const uint64_t need_r = 1 + (uint64_t)sd.nparts, need_s = 2 + ((uint64_t)sd.nparts + 1) / 2;
        if (c->part_cursor[rv.proc] + need_r > kPartHeapSlots || c->part_cursor[sd.proc] + need_s > kPartHeapSlots)
            return MPXA_ERR_NOMEM;
        const uint64_t ro = c->part_cursor[rv.proc];
        c->part_cursor[rv.proc] += need_r;
        const uint64_t so = c->part_cursor[sd.proc];     // (after: sender and receiver may share a heap)
        c->part_cursor[sd.proc] += need_s;
        if (sd.proc == c->proc) {                       // local sender end
            mpxa_request_t q = c->ppending[sd.idx];
            char *dst = nullptr;
            if (rv.proc == c->proc || c->nprocs == 1) {
                dst = c->ppending[rv.idx]->pbuf;
            } else if (rv.part_bytes) {
                const std::string key(rv.h.reserved, sizeof rv.h.reserved);
                auto it = c->ipc_opened.find({rv.proc, key});
                if (it == c->ipc_opened.end()) {
                    void *m = nullptr;
                    CK(cudaIpcOpenMemHandle(&m, rv.h, cudaIpcMemLazyEnablePeerAccess));
                    it = c->ipc_opened.emplace(std::make_pair(rv.proc, key), (char *)m).first;
                }
                dst = it->second + rv.buf_off;
            }
            q->sdev = mpxa_psend_dev_t{};
            q->sdev.src = (const unsigned char *)q->pbuf;
            q->sdev.dst = (unsigned char *)dst;
            q->sdev.part_bytes = q->part_bytes;
            q->sdev.n_parts = q->nparts;
            q->sdev.arr = pslot(c, rv.proc, ro + 1);
            q->sdev.cts = pslot(c, sd.proc, so + 1);
            q->sdev.scycle = pslot(c, sd.proc, so);
            q->sdev.done = (unsigned int *)pslot(c, sd.proc, so + 2);
            q->sdev.err = c->err_dev;
            q->sdev.timeout_ns = (long long)(c->timeout_s * 1e9);
            q->mycycle = pslot(c, sd.proc, so);
            q->readied.assign(q->nparts, 0);
            q->matched = true;
        }
        if (rv.proc == c->proc) {                       // local receiver end
            mpxa_request_t q = c->ppending[rv.idx];
            q->mycycle = pslot(c, rv.proc, ro);
            q->arr = pslot(c, rv.proc, ro + 1);
            q->cts_remote = pslot(c, sd.proc, so + 1);
            q->peer_nparts = sd.nparts;
            q->peer_part_bytes = sd.part_bytes;
            q->matched = true;
        }
    }
    c->ppending.clear();
    return MPXA_SUCCESS;
}

int mpxa_pready_range(mpxa_request_t q, int lo, int hi, mpxa_stream_t st) {
    if (!q || q->pkind != 1) return MPXA_ERR_ARG;
    if (!q->matched || !q->active) return MPXA_ERR_LIFECYCLE;
    if (lo < 0 || hi > q->nparts || lo >= hi) return MPXA_ERR_ARG;
    for (int i = lo; i < hi; i++)
        if (q->readied[i]) return MPXA_ERR_ARG;       // each partition once per cycle
    for (int i = lo; i < hi; i++) q->readied[i] = 1;
    cudaError_t e = launch_part_pready(q->sdev, lo, hi - lo, S(st));
    if (e != cudaSuccess) return MPXA_ERR_CUDA;
    q->comm->launches++;
    return MPXA_SUCCESS;
}

int mpxa_pready(mpxa_request_t q, int i, mpxa_stream_t st) { return mpxa_pready_range(q, i, i + 1, st); }

namespace {
// sender partitions covering receiver partitions [lo, hi) (byte intervals)
void cover(const mpxa_request_t q, int lo, int hi, int &a, int &b) {
    const uint64_t total = (uint64_t)q->nparts * q->part_bytes;
    const uint64_t blo = (uint64_t)lo * q->part_bytes, bhi = std::min(total, (uint64_t)hi * q->part_bytes);
    const uint64_t bs = q->peer_part_bytes;
    if (bs == 0 || blo >= bhi) { a = 0; b = q->peer_nparts; return; }   // zero-byte message: all flags
    a = (int)(blo / bs);
    b = (int)((bhi + bs - 1) / bs);
}
}  // namespace

int mpxa_parrived(mpxa_request_t q, int j, int *flag) {
    if (!q || !flag || q->pkind != 2) return MPXA_ERR_ARG;
    if (!q->matched || !q->active) return MPXA_ERR_LIFECYCLE;
    if (j < 0 || j >= q->nparts) return MPXA_ERR_ARG;
    int a, b;
    cover(q, j, j + 1, a, b);
    std::vector<unsigned long long> f((size_t)std::max(1, b - a));
    if (b > a) {
        CK(cudaMemcpyAsync(f.data(), q->arr + a, sizeof(unsigned long long) * (size_t)(b - a), cudaMemcpyDeviceToHost,
                           q->comm->pquery));
        CK(cudaStreamSynchronize(q->comm->pquery));
    }
    int ok = 1;
    for (int i = 0; i < b - a; i++) ok &= f[(size_t)i] >= q->cycle;
    *flag = ok;
    return MPXA_SUCCESS;
}

int mpxa_parrived_wait(mpxa_request_t q, int lo, int hi, mpxa_stream_t st) {
    if (!q || q->pkind != 2) return MPXA_ERR_ARG;
    if (!q->matched || !q->active) return MPXA_ERR_LIFECYCLE;
    if (lo < 0 || hi > q->nparts || lo >= hi) return MPXA_ERR_ARG;
    int a, b;
    cover(q, lo, hi, a, b);
    if (b > a) {
        cudaError_t e = launch_part_wait(q->arr, a, b, q->mycycle, q->comm->err_dev,
                                         (long long)(q->comm->timeout_s * 1e9), S(st));
        if (e != cudaSuccess) return MPXA_ERR_CUDA;
        q->comm->launches++;
    }
    return MPXA_SUCCESS;
}

int mpxa_psend_device(mpxa_request_t q, void *out, size_t bytes) {
    if (!q || !out || q->pkind != 1 || bytes < sizeof(mpxa_psend_dev_t)) return MPXA_ERR_ARG;
    if (!q->matched) return MPXA_ERR_LIFECYCLE;
    memcpy(out, &q->sdev, sizeof(mpxa_psend_dev_t));
    return MPXA_SUCCESS;
}

// ---- neighborhood collectives ------------------------------------------
int mpxa_dist_graph_create_adjacent(mpxa_comm_t c, const int *indegree, const int *sources, const int *sourceweights,
                                    const int *outdegree, const int *destinations, const int *destweights,
                                    const void *info, int reorder, mpxa_topo_t *topo) {
    (void)info; (void)reorder;
    if (!c || !topo || !indegree || !outdegree) return MPXA_ERR_ARG;
    *topo = nullptr;
    int64_t nin = 0, nout = 0;
    for (int t = 0; t < c->R; t++) {
        if (indegree[t] < 0 || outdegree[t] < 0) return MPXA_ERR_ARG;
        nin += indegree[t];
        nout += outdegree[t];
    }
    if ((nin && !sources) || (nout && !destinations)) return MPXA_ERR_ARG;
    for (int64_t e = 0; e < nin; e++) if (sources[e] < 0 || sources[e] >= c->p) return MPXA_ERR_ARG;
    for (int64_t e = 0; e < nout; e++) if (destinations[e] < 0 || destinations[e] >= c->p) return MPXA_ERR_ARG;
    std::unique_ptr<mpxa_topo_s> T(new mpxa_topo_s());
    T->comm = c;
    T->p = c->p;
    T->nin = nin;
    T->nout = nout;
    std::vector<int> zin((size_t)nin, 1), zout((size_t)nout, 1);
    int r = allgather_concat(c, indegree, (size_t)c->R, T->indeg);
    if (!r) r = allgather_concat(c, outdegree, (size_t)c->R, T->outdeg);
    if (!r) r = allgather_concat(c, sources, (size_t)nin, T->src);
    if (!r) r = allgather_concat(c, destinations, (size_t)nout, T->dst);
    if (!r) r = allgather_concat(c, sourceweights ? sourceweights : zin.data(), (size_t)nin, T->srcw);
    if (!r) r = allgather_concat(c, destweights ? destweights : zout.data(), (size_t)nout, T->dstw);
    if (r) return r;
    for (int q = 0; q < c->proc * c->R; q++) { T->in0 += T->indeg[q]; T->out0 += T->outdeg[q]; }
    *topo = T.release();
    return MPXA_SUCCESS;
}

int mpxa_topo_free(mpxa_topo_t *topo) {
    if (!topo || !*topo) return MPXA_ERR_ARG;
    delete *topo;
    *topo = nullptr;
    return MPXA_SUCCESS;
}

int mpxa_neighbor_alltoallv_init(const void *s, const int64_t *sc, const int64_t *sd, size_t sb, void *r,
                                 const int64_t *rc, const int64_t *rd, size_t rb, size_t w, mpxa_topo_t topo,
                                 const void *info, mpxa_request_t *req) {
    (void)info;
    if (!req) return MPXA_ERR_ARG;
    *req = nullptr;
    return neighbor_impl(false, s, sc, sd, sb, r, rc, rd, rb, w, nullptr, nullptr, topo, nullptr, req);
}

int mpxa_neighbor_alltoallv_locality_init(const void *s, const int64_t *sc, const int64_t *sd, size_t sb, void *r,
                                          const int64_t *rc, const int64_t *rd, size_t rb, size_t w,
                                          const int64_t *sidx, const int64_t *ridx, mpxa_topo_t topo,
                                          const void *info, mpxa_request_t *req) {
    (void)info;
    if (!req) return MPXA_ERR_ARG;
    *req = nullptr;
    return neighbor_impl(true, s, sc, sd, sb, r, rc, rd, rb, w, sidx, ridx, topo, nullptr, req);
}

int mpxa_neighbor_alltoallv(const void *s, const int64_t *sc, const int64_t *sd, size_t sb, void *r,
                            const int64_t *rc, const int64_t *rd, size_t rb, size_t w, mpxa_topo_t topo,
                            mpxa_stream_t st) {
    return neighbor_impl(false, s, sc, sd, sb, r, rc, rd, rb, w, nullptr, nullptr, topo, S(st), nullptr);
}

// ---- registry / selector -----------------------------------------------------------------
int mpxa_set_algorithm(mpxa_comm_t c, mpxa_op_t op, mpxa_algo_t a) {
    if (!c || op < 0 || op > 2) return MPXA_ERR_ARG;
    if (a != MPXA_ALGO_DEFAULT && !algo_valid(op, a)) return MPXA_ERR_ALGO;
    c->user_algo[op] = a;
    return MPXA_SUCCESS;
}

int mpxa_get_algorithm(mpxa_comm_t c, mpxa_op_t op, size_t bytes, mpxa_algo_t *chosen) {
    if (!c || !chosen || op < 0 || op > 2) return MPXA_ERR_ARG;
    *chosen = (mpxa_algo_t)default_algo(c, op, bytes);
    return MPXA_SUCCESS;
}

int mpxa_list_algorithms(mpxa_op_t op, mpxa_algo_t *out, int *n) {
    if (!n || op < 0 || op > 3) return MPXA_ERR_ARG;
    static const mpxa_algo_t a2a[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_BRUCK, MPXA_ALGO_HIER};
    static const mpxa_algo_t a2av[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_HIER, MPXA_ALGO_BRUCK};
    static const mpxa_algo_t ag[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_BRUCK, MPXA_ALGO_RING, MPXA_ALGO_HIER};
    static const mpxa_algo_t nb[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_LOCALITY};
    const mpxa_algo_t *src = op == 0 ? a2a : op == 1 ? a2av : op == 2 ? ag : nb;
    int cnt = op == 3 ? 2 : op == 2 ? 4 : 3;
    if (out) {
        if (*n < cnt) { *n = cnt; return MPXA_ERR_ARG; }
        for (int i = 0; i < cnt; i++) out[i] = src[i];
    }
    *n = cnt;
    return MPXA_SUCCESS;
}

int mpxa_load_selector(mpxa_comm_t c, const char *path) {
    if (!c || !path) return MPXA_ERR_ARG;
    return load_selector_file(c, path);
}

int mpxa_config_digest(mpxa_comm_t c, uint64_t *digest) {
    if (!c || !digest) return MPXA_ERR_ARG;
    *digest = knob_digest(c, c->heap0);
    return MPXA_SUCCESS;
}

}  // extern "C"

namespace {
int load_selector_file(mpxa_comm_t c, const char *path) {
    std::ifstream f(path);
    if (!f) return MPXA_ERR_ARG;
    std::vector<SelEntry> t;
    std::string line;
    while (std::getline(f, line)) {
        auto h = line.find('#');
        if (h != std::string::npos) line = line.substr(0, h);
        std::stringstream ss(line);
        std::vector<std::string> tok;
        for (std::string x; ss >> x;) tok.push_back(x);
        if (tok.empty()) continue;
        // "op p R max_bytes algo" (any GPU count / group) or "op p R G g max_bytes algo"
        if (tok.size() != 5 && tok.size() != 7) return MPXA_ERR_ARG;
        const bool full = tok.size() == 7;
        const std::string &op = tok[0], &algo = tok.back();
        SelEntry e{};
        char *endp = nullptr;
        e.p = (int)strtol(tok[1].c_str(), &endp, 10);
        e.R = (int)strtol(tok[2].c_str(), &endp, 10);
        e.G = full ? (int)strtol(tok[3].c_str(), &endp, 10) : -1;
        e.g = full ? (int)strtol(tok[4].c_str(), &endp, 10) : -1;
        const unsigned long long mb = strtoull(tok[full ? 5 : 3].c_str(), &endp, 10);
        e.op = op == "alltoall" ? 0 : op == "alltoallv" ? 1 : op == "allgather" ? 2 : -1;
        e.algo = algo == "pairwise" ? 1 : algo == "bruck" ? 2 : algo == "hier" ? 3 : algo == "ring" ? 4 : 0;
        e.max_bytes = mb;
        if (e.op < 0 || !algo_valid(e.op, e.algo)) return MPXA_ERR_ARG;
        t.push_back(e);
    }
    c->selector = t;
    return MPXA_SUCCESS;
}
}  // namespace

extern "C" {

// ---- host-only plan introspection (include/mpxa_plan.h) ---------------------------------
int mpxa_plan_build(int op, int algo, int p, int R, int G, int g, int stop_stage, const int64_t *cnt,
                    const int64_t *sd, const int64_t *rd, void **plan) {
    if (!plan) return MPXA_ERR_ARG;
    *plan = nullptr;
    auto P = new Program();
    bool ok = false;
    const char *hs = getenv("MPXA_HIER_STAGED");   // same knob as the comms (tests of both forms)
    const bool staged = hs && atoi(hs) != 0;
    if (op == MPXA_OP_ALLTOALL) ok = build_alltoall(*P, algo, p, R, G, g, stop_stage, staged);
    else if (op == MPXA_OP_ALLGATHER) ok = build_allgather(*P, algo, p, R, G, stop_stage, g);
    else if (op == MPXA_OP_ALLTOALLV && cnt && sd && rd) ok = build_alltoallv(*P, algo, p, R, G, g, cnt, sd, rd, staged);
    if (!ok) { delete P; return MPXA_ERR_ALGO; }
    *plan = P;
    return MPXA_SUCCESS;
}

int mpxa_plan_build_neighbor(int p, int R, int G, int g, int locality, const int *indeg, const int *src,
                             const int64_t *rc, const int64_t *rd, const int *outdeg, const int *dst,
                             const int64_t *sc, const int64_t *sd, const int64_t *send_idx,
                             const int64_t *recv_idx, void **plan) {
    if (!plan || !indeg || !outdeg) return MPXA_ERR_ARG;
    *plan = nullptr;
    auto P = new Program();
    const char *hs = getenv("MPXA_HIER_STAGED");   // same knob as the comms
    int r = build_neighbor(*P, locality != 0, p, R, G, g, indeg, src, rc, rd, outdeg, dst, sc, sd, send_idx, recv_idx,
                           hs && atoi(hs) != 0);
    if (r) { delete P; return r; }
    *plan = P;
    return MPXA_SUCCESS;
}

int mpxa_plan_eager(const void *plan, size_t unit, void **eager) {
    if (!plan || !eager || unit == 0) return MPXA_ERR_ARG;
    *eager = nullptr;
    const Program *P = (const Program *)plan;
    if (P->G < 2) return MPXA_ERR_ALGO;
    auto Q = new Program();
    if (!build_ll(*P, unit, P->p / P->G, *Q)) { delete Q; return MPXA_ERR_ALGO; }
    *eager = Q;
    return MPXA_SUCCESS;
}

int mpxa_plan_info(const void *plan, mpxa_plan_info_t *info) {
    if (!plan || !info) return MPXA_ERR_ARG;
    const Program *P = (const Program *)plan;
    info->nsteps = P->nsteps();
    info->work_units = P->work_units;
    info->max_move = P->max_move;
    info->max_step_units = P->max_step_units;
    info->signals = P->signals;
    int64_t tm = 0;
    for (auto &m : P->moves) tm += (int64_t)m.size();
    info->total_moves = tm;
    info->nflows = P->nflows;
    info->max_step_moves = P->max_step_moves;
    return MPXA_SUCCESS;
}

int mpxa_plan_steps(const void *plan, int gpu, mpxa_plan_step *out, int *n) {
    if (!plan || !n) return MPXA_ERR_ARG;
    const Program *P = (const Program *)plan;
    if (gpu < 0 || gpu >= P->G) return MPXA_ERR_ARG;
    const auto &v = P->steps[gpu];
    if (out) {
        if (*n < (int)v.size()) return MPXA_ERR_ARG;
        static_assert(sizeof(mpxa_plan_step) == sizeof(Step), "plan step layout");
        memcpy(out, v.data(), sizeof(Step) * v.size());
    }
    *n = (int)v.size();
    return MPXA_SUCCESS;
}

int mpxa_plan_moves(const void *plan, int gpu, mpxa_plan_move *out, int *n) {
    if (!plan || !n) return MPXA_ERR_ARG;
    const Program *P = (const Program *)plan;
    if (gpu < 0 || gpu >= P->G) return MPXA_ERR_ARG;
    const auto &v = P->moves[gpu];
    if (out) {
        if (*n < (int)v.size()) return MPXA_ERR_ARG;
        static_assert(sizeof(mpxa_plan_move) == sizeof(Move), "plan move layout");
        memcpy(out, v.data(), sizeof(Move) * v.size());
    }
    *n = (int)v.size();
    return MPXA_SUCCESS;
}

// undocumented test hook: the execution path of the comm's last collective launch, as bits
// 1 small kernel, 2 eager (LL), 4 variable pieces, 8 dynamic work queues, 16 row-barrier
// sync, 32 owned flows, 64 WORK in shared memory, 128 warp-ring dynamic mode, 256 tiny kernel
int mpxa__last_launch(mpxa_comm_t c, uint32_t *bits) {
    if (!c || !bits) return MPXA_ERR_ARG;
    *bits = c->last_path;
    return MPXA_SUCCESS;
}

// undocumented debug hook (MPXA_TRACE builds): copy the device phase stamps
int mpxa__trace(mpxa_comm_t c, uint64_t *out16) {
    if (!c || !out16) return MPXA_ERR_ARG;
    CK(cudaMemcpy(out16, (char *)c->dc + offsetof(DevComm, trace), 32 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return MPXA_SUCCESS;
}

int mpxa_plan_free(void *plan) {
    delete (Program *)plan;
    return MPXA_SUCCESS;
}

}  // extern "C"

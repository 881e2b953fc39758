#pragma once
// libmpxa host runtime, internal header: the communicator / request / topology records, the
// program cache types and launch-sizing constants, and the functions the runtime's files share
// (comm.cpp, launch.cpp, collectives.cpp, partitioned.cpp, selector.cpp, plan_api.cpp).  Not
// part of the C ABI (include/mpxa.h).
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

namespace mpxa_rt {

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
constexpr uint64_t kWringMinPiece = 16u << 10;  // warp rings: smallest queue piece (4 / 8 KiB: slower)
constexpr uint64_t kWringFloorVol20 = 192ull << 20, kWringFloorVol24 = 256ull << 20;   // warp rings: larger
                                                 // piece floors (20 / 24 KiB) from these busiest-GPU volumes
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


}  // namespace mpxa_rt
using namespace mpxa_rt;

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
    int prefetch = 1;                         // MPXA_NO_PREFETCH=1: no pre-wait L2 prefetch (dynamic mode)
    int wslack = 3;                           // MPXA_WSLACK: warp-ring stages kept out of the load window
                                              // (measured, cfg4 p = 8 int64 / int32, means 1-8 MiB, seeds 0-1:
                                              // 3 loads in flight at or below 4 (wslack 2) in all 16 cases, 0.1-1 us;
                                              // 2 loads slower from 2 MiB, 1 load +25 %: profiles/r02/cfg4_wslack_s18.txt)
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

namespace mpxa_rt {

// comm.cpp: bootstrap, symmetric memory
bool dtype_ok(size_t w);
int h2d_complete(void *dst, const void *src, size_t n);
int bootstrap(mpxa_comm_t c, const void *in, void *out, size_t bytes);
int allgather_var(mpxa_comm_t c, const void *mine, size_t n, std::vector<std::vector<char>> &out);
int ipc_exchange(mpxa_comm_t c, void *local, char **mapped);
int upload_tables(mpxa_comm_t c);
int ensure_work(mpxa_comm_t c, size_t need_per_gpu);

// comm.cpp: knobs
void read_knobs(mpxa_comm_t c);
uint64_t knob_digest(mpxa_comm_t c, size_t heap);

// launch.cpp: programs
void prog_facts(DevProg &dp);
size_t serialize(const Program &P, std::vector<char> &buf, uintptr_t dbase);
size_t serialized_size(const Program &P);

// launch.cpp: program cache, launch decisions
bool build_ll(const Program &P, uint64_t unit, int R, Program &Q, int64_t max_words = kLLWords);
void prebuild_companions(mpxa_comm_t c, const DevProg &dp, uint64_t unit);
int upload_program(const Program &P, std::shared_ptr<DevProg> &out);
int var_program(const DevProg &dp, int64_t chop, const DevProg *&out);
int cached_uniform(mpxa_comm_t c, int op, int algo, int stage, std::shared_ptr<DevProg> &out);
uint64_t cdiv(uint64_t a, uint64_t b);
Grid choose_grid(mpxa_comm_t c, const Program &P, uint64_t unit);
int make_params(mpxa_comm_t c, ExecParams &E, const DevProg &dp, const char *send, char *recv,
                uint64_t unit, uint64_t send_stride, uint64_t recv_stride);
int run_program(mpxa_comm_t c, const DevProg &dp, const char *send, char *recv, uint64_t unit,
                uint64_t send_stride, uint64_t recv_stride, cudaStream_t stream, const Grid *grid = nullptr,
                bool pdl = true);
int run_dynamic(mpxa_comm_t c, const Program &P, const char *send, char *recv, uint64_t unit,
                uint64_t send_stride, uint64_t recv_stride, cudaStream_t stream);

// selector.cpp
int default_algo(mpxa_comm_t c, int op, size_t bytes);
bool algo_valid(int op, int algo);

// selector.cpp
int load_selector_file(mpxa_comm_t c, const char *path);

// collectives.cpp: argument checks and implementations
inline cudaStream_t S(mpxa_stream_t s) { return (cudaStream_t)s; }
bool overlap(const void *a, size_t na, const void *b, size_t nb);
int check_uniform(mpxa_comm_t c, const void *send, size_t count, size_t w, void *recv, int op);
int host_view(const int64_t *&a, size_t n, std::vector<int64_t> &store, cudaStream_t stream);
int gather_v(mpxa_comm_t c, const int64_t *sc, const int64_t *sd, const int64_t *rc,
             const int64_t *rd, size_t w, size_t send_bpr, size_t recv_bpr,
             std::vector<int64_t> &C, std::vector<int64_t> &SD, std::vector<int64_t> &RD, cudaStream_t stream);
uint64_t fnv(uint64_t h, const void *p, size_t n);
int vprogram(mpxa_comm_t c, int algo, const std::vector<int64_t> &C, const std::vector<int64_t> &SD,
             const std::vector<int64_t> &RD, mpxa_comm_s::VEntry *&out);
int alltoallv_impl(const void *sendbuf, const int64_t *sc, const int64_t *sd, size_t send_bpr,
                   void *recvbuf, const int64_t *rc, const int64_t *rd, size_t recv_bpr, size_t w,
                   int algo, mpxa_comm_t c, cudaStream_t stream, mpxa_request_t *req);
int uniform_impl(int op, const void *sendbuf, size_t count, size_t w, void *recvbuf, int algo,
                 mpxa_comm_t c, cudaStream_t stream, mpxa_request_t *req, int stage = -1,
                 bool force_bruck = false);
int neighbor_impl(bool locality, const void *sendbuf, const int64_t *sc, const int64_t *sd, size_t send_bpr,
                  void *recvbuf, const int64_t *rc, const int64_t *rd, size_t recv_bpr, size_t w,
                  const int64_t *sidx, const int64_t *ridx, mpxa_topo_t topo, cudaStream_t stream,
                  mpxa_request_t *req);

template <typename T>
int allgather_concat(mpxa_comm_t c, const T *mine, size_t n, std::vector<T> &out) {
    std::vector<std::vector<char>> parts;
    int rc = allgather_var(c, mine, n * sizeof(T), parts);
    if (rc) return rc;
    out.clear();
    for (auto &b : parts) out.insert(out.end(), (const T *)b.data(), (const T *)(b.data() + b.size()));
    return MPXA_SUCCESS;
}

}  // namespace mpxa_rt

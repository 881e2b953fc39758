// Internal types shared by the host runtime (comm.cpp, launch.cpp, collectives.cpp, partitioned.cpp, plan.cpp, ...) and the sm_100a
// kernels (exec_kernel.cu, small_kernels.cu, aux_kernels.cu).  Not part of the C ABI (include/mpxa.h).
//
// Execution model: every collective call is compiled, on the host, into a
// PROGRAM per GPU: a list of STEPS, each a list of MOVES (byte copies between rank
// buffers, possibly on a peer GPU).  One kernel launch executes the whole program.  CTA c
// of a GPU owns "column slice" c of every unit (block / segment) that moves, through all
// steps, so a step's inputs written by this GPU were written by the same CTA and only a
// __syncthreads separates steps; inputs written by a peer GPU were written by the peer's
// CTA c, which signals a per-(src GPU, CTA) flag that this CTA acquires.  No grid-wide
// barrier is ever needed.
#pragma once
#include <stdint.h>

namespace mpxa {

constexpr int kMaxGpus = 32;       // processes or virtual GPUs per comm (signal masks are 32-bit)
constexpr int kMaxCtas = 1024;     // CTAs per GPU per launch (flag slots per source GPU)
#ifndef MPXA_THREADS
#define MPXA_THREADS 128
#endif
constexpr int kThreads = MPXA_THREADS;   // threads per CTA of the executor kernel (warp 0: TMA producer;
                                         // 128: no register spills at 2 CTAs / SM, measured fastest)
// TMA ring configurations (runtime-selected per launch):
//   mid : 6 x 16 KiB stages, 2 CTAs / SM  (many CTAs: mid-size messages, latency)
//   big : 6 x 32 KiB stages, 1 CTA / SM   (more bytes in flight per SM: large messages)
constexpr int kMaxStages = 8;
struct TmaConfig {
    int stages, chunk, ahead;
};
constexpr int kRingStages = 6;   // both configurations' stage count (the producer's ring index)
constexpr TmaConfig kTmaMid = {kRingStages, 16384, 4};
constexpr TmaConfig kTmaBig = {kRingStages, 32768, 4};
constexpr int kMaxDynSmem = 6 * 32768;
constexpr int kMoveTile = kThreads;   // moves staged in shared memory at a time (one per thread)
constexpr int kMaxDynTiles = 64;      // dynamic mode: move tiles per step (queues per tile)
constexpr int kMaxStepsSmem = 64;     // step tables kept in shared memory by the kernels
// warp-ring dynamic mode (ExecParams::wring): every warp of the CTA is its own TMA pipeline
// over a ring of kWStages stages of kWChunk bytes (same 96 KiB of dynamic shared memory as
// the mid ring, so 2 CTAs / SM); moves that are not 16-B congruent are stored by the warp
// with 16-B stores shifted out of shared memory instead of through LSU registers
constexpr int kWarpsExec = kThreads / 32;
constexpr int kWStages = 6;
constexpr int kWChunk = 4096;
constexpr uint64_t kSmallKernelMax = 8192;  // longest move (bytes) the small-message kernel takes
constexpr int kSmallMovesSmem = 4096;       // program moves cached in shared memory by the small kernel
enum { kSmallCommon = 0, kSmallVar = 1, kSmallLocal = 2, kSmallLL = 3 };   // small-kernel instantiations
constexpr int kSmallWorkSmem = 48 << 10;    // kSmallLocal: WORK rows in shared memory up to this size
                                            // (+ 4096 cached moves + static smem <= 227 KiB)
constexpr int kRankTable = 256;   // small kernel: per-rank buffer bases kept in shared memory
constexpr int kMaxWindows = 16;    // registered recv windows per process

enum BufKind : uint8_t { BK_SEND = 0, BK_RECV = 1, BK_WORK = 2,
                         BK_LL = 3 };   // eager (LL) staging word stream: rank = peer GPU, offset in words

// One copy of `len` units from (src_kind, src_rank, src_off) to (dst_kind, dst_rank, dst_off).
// Offsets and lengths are in UNITS of ExecParams::unit bytes.  fanout = 1: copy to the
// dst_kind buffer of EVERY rank at dst_off (allgather direct); dst_rank is ignored.
// flow: identity of the data the move carries (its origin block / segment), preserved
// along the data's path through the steps; CTAs own (flow group, column slice) pairs.
struct Move {
    int64_t src_off;
    int64_t dst_off;
    int64_t len;
    uint32_t flow;
    uint16_t src_rank;
    uint16_t dst_rank;
    uint8_t src_kind;
    uint8_t dst_kind;
    uint8_t fanout;
    uint8_t pad[5];
};
static_assert(sizeof(Move) == 40, "Move layout");

// Moves of a step are sorted by flow; findex[flow_index + x] = number of the step's moves
// with flow < x (x = 0..nflows), so flow group [x0, x1) owns moves [findex[x0], findex[x1]).
struct Step {
    int32_t move_begin;     // [move_begin, move_end) in the GPU's move array
    int32_t move_end;
    uint32_t signal_mask;   // remote GPUs this GPU writes to in this step
    uint32_t wait_mask;     // remote GPUs that write into this GPU in this step
    int64_t total_len;      // sum of move lengths in units (host-side sizing)
    int64_t max_len;        // max move length in units (host-side path hints)
    int32_t flow_index;     // offset of this step's flow index in GpuProg::findex
    int32_t dense_base;     // >= 0: move k of the step carries flow dense_base + k (the flow
                            // index is then arithmetic: no findex lookup); -1 otherwise
};
static_assert(sizeof(Step) == 40, "Step layout");

struct GpuProg {
    const Step *steps;
    const Move *moves;
    const int32_t *findex;
    int32_t nsteps;
    int32_t nmoves;
};

// Clear-to-send message from receiver GPU d to sender GPU s, stored in s's region.
struct CtsSlot {
    uint64_t epoch;         // written last, with release semantics
    uint64_t win;           // registered window of d's recvbuf (recv_from_cts mode)
    uint64_t off;           // byte offset of d's recvbuf in that window
    uint64_t pad;
};

// Per-GPU symmetric region (device memory, IPC-exported in multi-process mode).
constexpr int kLLWords = 32768;     // eager staging words per (parity, source GPU): 128 KiB payload
struct SymRegion {
    CtsSlot cts[kMaxGpus];                    // cts[d]: receiver d cleared this GPU to send
    uint64_t flags[kMaxGpus][kMaxCtas];       // flags[s][c]: src GPU s, CTA c, (epoch<<8)|(step+1)
    // eager (LL) mode: ll[seq & 1][s][w] = (seq << 32) | 4 payload bytes from source GPU s --
    // the flag travels in every 8-byte word, so no fence or separate signal is needed; the
    // parity alternates per eager launch (SURVEY §8 A9 "epoch-parity staging")
    uint64_t ll[2][kMaxGpus][kLLWords];
};

// Per-communicator device-resident state (rewritten by the host only between launches:
// heap growth, buffer registration).  epoch/done make the launch sequence number
// device-side, so a captured CUDA graph replays with fresh epochs.
struct DevComm {
    char *work_base[kMaxGpus];              // per GPU: workspace heap (mapped here)
    SymRegion *sym[kMaxGpus];               // per GPU: symmetric region (mapped here)
    char *win_table[kMaxGpus * kMaxWindows];  // per GPU: registered recv windows (mapped here)
    uint64_t epoch;                         // epochs completed on this GPU (or emulated set)
    uint32_t done_ctas;                     // CTAs of the current launch that finished
    uint32_t pad;
    uint32_t dyn_next[kMaxGpus * kMaxDynTiles];   // work-queue heads of dynamic launches, per (GPU
    uint32_t dyn_next2[kMaxGpus * kMaxDynTiles];  // row, move tile): TMA pieces / LSU pieces;
                                                  // reset by the launch's last CTA
    uint32_t dyn_bar[kMaxGpus];                   // multi-step dynamic mode: per-row step barrier
    uint64_t ll_seq;                        // eager (LL) launches completed (flag of the next + 1)
    uint64_t trace[32];                     // MPXA_TRACE builds: %globaltimer phase stamps
};

// Launch parameters (~130 B).  Buffers are the caller's process-level rank-major buffers.
struct ExecParams {
    const GpuProg *progs;      // device array [G] (only progs[my_gpu] used in multi-process)
    GpuProg prog;              // modes 0 and 2: this GPU's program by value (saves a round trip)
    DevComm *dc;
    const char *send;          // this process's sendbuf (first local rank)
    char *recv;                // this process's recvbuf
    uint64_t unit;             // bytes per unit
    uint64_t send_stride;      // bytes between consecutive local ranks' buffers
    uint64_t recv_stride;
    uint64_t work_stride;
    uint64_t recv_win;         // multi-process: registered window of recv, and its offset
    uint64_t recv_off;
    int32_t *err;              // host-mapped error word (watchdog)
    int64_t timeout_ns;
    int32_t G;                 // GPUs (processes or virtual)
    int32_t R;                 // ranks per GPU
    int32_t p;                 // ranks
    int32_t my_gpu;            // -1: emulated, GPU = blockIdx.y
    int32_t nflows;            // flows of the program (same on every GPU)
    int32_t nS;                // column slices per move; CTA c owns slice c % nS
    int32_t nF;                // flow groups; CTA c owns flow group c / nS
    int32_t mode;              // 0 single GPU, 1 emulated GPUs, 2 multi-process
    int32_t stages;            // TMA ring: stages x chunk bytes of dynamic shared memory
    int32_t chunk;
    int32_t ahead;             // loads in flight ahead of the oldest store (<= stages - 2)
    int32_t small_ppm;         // small kernel: 16-byte pieces per move (ceil(max move / 16))
    int32_t small_cache;       // small kernel: moves cached in shared memory (0 = read global)
    int32_t d0_base;           // step 0 dense (Step::dense_base >= 0): its base flow, and
    int32_t d0_n;              // its move count -> step 0's moves are fetched in the prologue
    // dynamic mode (dyn_units = number of move tiles > 0): single-step program whose moves are
    // cut into pieces of at most dyn_u bytes that CTAs take from device work queues
    // (DevComm::dyn_next) -- per-SM bandwidth differs across the chip, so static slices
    // leave a tail of slow CTAs
    int32_t dyn_units;         // queue tiles used by the launch (all steps)
    int32_t dyn_u;
    int32_t small_a16;         // every local offset, length, base and stride is a 16-B multiple
    int32_t small_own;         // small kernel, multi-step on several CTAs without barriers: CTA c
                               // moves the flows f with f % small_own == c in every step (same
                               // owner across steps -> __syncthreads suffices); 0 = off
    int32_t small_var;         // small kernel: moves of very different lengths -- pieces counted
                               // exactly per tile of moves (block scan) instead of max-move slots
    int32_t small_swork;       // small kernel, one CTA on one GPU, moves resolved (kSmallLocal): the
                               // WORK rows live in this CTA's dynamic shared memory after the
                               // cached moves, so steps chain through shared memory
    int32_t small_threads;     // small kernel block size (0 = 512); >= p, >= nsteps
    int32_t dyn_sync;          // multi-step dynamic mode: steps separated by a per-GPU-row CTA
                               // barrier and ONE flag per peer GPU (slot 0), so any CTA may move
                               // any piece (no flow ownership needed)
    int32_t small_ll;          // small kernel, eager (LL) companion program: moves to peer GPUs
                               // are word streams into their staging (BK_LL); each step lists
                               // its receive moves last (Step::wait_mask = their number)
    int32_t wring;             // dynamic mode with per-warp TMA rings (kWStages x kWChunk each);
                               // stages / chunk then describe the whole dynamic smem
    int32_t small_a8;          // small kernel: every local offset, length, base and stride is an
                               // 8-B multiple (not all 16): pieces move as 8-byte words
    int32_t wslack;            // warp-ring mode: stages kept out of the load window (1..kWStages-1; 3)
    int32_t small_a4;          // tiny kernel: every offset, length, base and stride a 4-B multiple
                               // (not all 8): pieces move as 4-byte words, no funnel shifts
    int32_t tiny_step_items;   // tiny multi-step kernel: 16-B pieces of the busiest step (launch
                               // choice of the one-piece-per-thread build)
    int32_t dyn_prefetch;      // dynamic mode, one GPU: the grid's first pieces (this many per CTA)
                               // prefetched into L2 before the dependency wait
};

}  // namespace mpxa

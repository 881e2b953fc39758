/*
 * mpxa.h -- C ABI of the B200-native MPI Advance collectives hot path
 * (arXiv 2309.07337, "MPI Advance: Open-Source Message Passing Optimizations").
 *
 * What the calls compute (the paper adopts MPI semantics: MPIX_Alltoallv is a drop-in
 * for MPI_Alltoallv, §2.1):
 *   alltoall : recv_r[j] = send_j[r]                    (personalized exchange)
 *   alltoallv: recv_r[rdispls_r[j]*w, +recvcounts_r[j]*w) = send_j[sdispls_j[r]*w, +..)
 *   allgather: recv_r[j] = send_j                        (concatenation in rank order)
 * in the paper's algorithm families ("minimize message count for small data
 * sizes and bytes transported for larger messages"; "distinguishing between inter- and
 * intra- node communication"): pairwise/direct exchange, Bruck's log-step algorithm
 * (local rotation, bit-indexed block send/recv, inverse rotation), ring, and the
 * locality-aware hierarchical variant (gather within a group, exchange once between
 * groups, redistribute).  Every implementation is public and selectable, with a default
 * ("make all implementations publicly available"); persistent forms follow
 * the MPI-4 init/start/wait model ("setup costs to be incurred
 * only once in the initialization method").
 *
 * Conventions
 *  - Every call returns an int status (mpxa_status); the library never aborts or throws
 *    across the ABI.  All argument errors are detected before any data moves.
 *  - Ranks: p = nprocs * ranks_per_proc logical ranks; rank r lives on process/GPU
 *    r / ranks_per_proc (contiguous map).  A process hosting R > 1 ranks
 *    passes PROCESS-LEVEL buffers laid out rank-major: [R][per-rank buffer].  Per-rank
 *    strides: alltoall send/recv p*count*w; allgather send count*w, recv p*count*w;
 *    alltoallv send_bytes_per_rank / recv_bytes_per_rank.  Count/displacement arrays of
 *    the v-form are R*p int64 (one row of p per local rank), in ELEMENTS of dtype_size.
 *  - Buffers (sendbuf, recvbuf) are DEVICE pointers on the comm's device.  Payload bytes
 *    are opaque (no datatype conversion; NaN payloads survive bit-exactly).  sendbuf and
 *    recvbuf must not overlap (no MPI_IN_PLACE).  Count/displacement arrays are HOST
 *    pointers unless stated otherwise.
 *  - Streams: `stream` is a cudaStream_t passed as void*.  Calls are stream-ordered:
 *    sendbuf must be ready in stream order and recvbuf is valid once the stream passes the
 *    call (one-shot) or mpxa_wait (persistent).  No call synchronizes the host with the
 *    device except where documented.
 *  - Ownership: the caller owns user buffers and streams; the library owns comms,
 *    requests, its device workspace (symmetric heap), flags and IPC mappings.
 *  - Collective calls (every process, same order): mpxa_init, mpxa_finalize,
 *    mpxa_register, every mpxa_alltoall* / mpxa_allgather* call, every *_init,
 *    mpxa_start and mpxa_request_free.  A ragged call order is erroneous and surfaces as
 *    MPXA_ERR_TIMEOUT from the device watchdog, not as a hang.
 *  - Multi-process mode (nprocs > 1): one process per GPU; recvbufs written by peers
 *    must lie in buffers registered with mpxa_register (or bound by a persistent *_init).
 *  - Completion across GPUs: large launches write peers' recvbufs
 *    directly after a clear-to-send from each receiver and release a flag per step; small
 *    launches (<= 128 KiB per GPU pair) run EAGER: the payload travels as 8-byte words that
 *    each carry the launch's sequence number into the receiver's staging (two parities,
 *    alternating per eager launch), the receiver copies it out -- no clear-to-send, no
 *    fence.  MPXA_NO_LL=1 disables eager mode.  Persistent requests build their eager form
 *    at *_init; one-shot calls build it on the first launch of a schedule for a dtype size,
 *    and if that first launch is inside a CUDA-graph capture it uses the direct protocol
 *    instead -- so in multi-process mode either every process or none captures the first
 *    one-shot call of a schedule (persistent requests have no such constraint).
 */
#ifndef MPXA_H
#define MPXA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpxa_comm_s *mpxa_comm_t;        /* MPIX_Comm analog */
typedef struct mpxa_request_s *mpxa_request_t;  /* MPIX_Request analog */
typedef void *mpxa_stream_t;                    /* a cudaStream_t (0 = legacy default)    */

typedef enum {
    MPXA_SUCCESS = 0,
    MPXA_ERR_ARG = 1,        /* NULL pointer, overlap, displ+count beyond capacity, negative
                                count, dtype_size not in {1,2,4,8,16}, bad stage index      */
    MPXA_ERR_ALGO = 2,       /* unknown / unsupported variant for this op or p */
    MPXA_ERR_LIFECYCLE = 3,  /* start on ACTIVE, wait on INACTIVE, free while ACTIVE */
    MPXA_ERR_TOPOLOGY = 4,   /* p not divisible by g, bad rank map / device */
    MPXA_ERR_MISMATCH = 5,   /* cross-process argument mismatch detected at *_init          */
    MPXA_ERR_CUDA = 6,       /* a CUDA runtime call failed                                    */
    MPXA_ERR_TIMEOUT = 7,    /* device watchdog fired; the comm is poisoned                   */
    MPXA_ERR_NOMEM = 8,      /* device or host allocation failed                              */
    MPXA_ERR_UNREGISTERED = 9 /* multi-process: recvbuf not in a registered buffer            */
} mpxa_status;

typedef enum { MPXA_OP_ALLTOALL = 0, MPXA_OP_ALLTOALLV = 1, MPXA_OP_ALLGATHER = 2,
               MPXA_OP_NEIGHBOR_ALLTOALLV = 3 } mpxa_op_t;

/* Variant registry.  PAIRWISE is the direct exchange
 * (for allgather: every rank pushes its block to every rank). */
typedef enum {
    MPXA_ALGO_DEFAULT = 0,   /* selector decides (mpxa_get_algorithm)                    */
    MPXA_ALGO_PAIRWISE = 1,  /* alltoall, alltoallv, allgather                            */
    MPXA_ALGO_BRUCK = 2,     /* alltoall, allgather, alltoallv (variable blocks)          */
    MPXA_ALGO_HIER = 3,      /* alltoall, alltoallv, allgather (groups of group_size ranks) */
    MPXA_ALGO_RING = 4,      /* allgather                                                 */
    MPXA_ALGO_LOCALITY = 5   /* neighbor alltoallv with global-index dedup    */
} mpxa_algo_t;

/* Adjacency topology (MPIX_Dist_graph_create_adjacent). */
typedef struct mpxa_topo_s *mpxa_topo_t;

/* Bootstrap callback: all-gather `bytes` bytes from every process into out[nprocs*bytes]
 * (out is ordered by process index).  Returns 0 on success.  Used only by collective
 * setup calls (init, register, *_init, heap growth), never on the data path. */
typedef int (*mpxa_allgather_fn)(const void *in, void *out, size_t bytes, void *ctx);

typedef struct {
    int nprocs;               /* processes (one per GPU)                                     */
    int proc;                 /* this process's index                                        */
    int ranks_per_proc;       /* R >= 1 logical ranks hosted by this process                 */
    int device;               /* CUDA device ordinal of this process                         */
    int group_size;           /* g for MPXA_ALGO_HIER; 0 -> R when R > 1, else 1             */
    int emulate_gpus;         /* nprocs == 1 only: run the multi-GPU protocol (flags, CTS,
                                 peer-style stores) over this many virtual GPUs of the one
                                 device in a cooperative launch; 0 or 1 = off                */
    mpxa_allgather_fn bootstrap_allgather;  /* required when nprocs > 1                      */
    void *ctx;                /* passed to bootstrap_allgather                               */
    size_t heap_bytes;        /* initial device workspace per process (0 = 64 MiB); grows
                                 collectively on demand                                      */
    double timeout_s;         /* device watchdog for flag waits (0 = 60 s)                   */
} mpxa_init_args;

/* ---- communicator (MPIX_Comm_init) ----------------- */
int mpxa_init(mpxa_comm_t *comm, const mpxa_init_args *args);
int mpxa_finalize(mpxa_comm_t comm);
int mpxa_comm_size(mpxa_comm_t comm, int *p);              /* total logical ranks p          */
int mpxa_comm_rank0(mpxa_comm_t comm, int *first_rank);    /* first rank hosted here         */
/* Returns MPXA_ERR_TIMEOUT if the device watchdog has fired on this comm (call after the
 * stream has been synchronized), else MPXA_SUCCESS.  Local. */
int mpxa_comm_check(mpxa_comm_t comm);
/* Number of kernels this comm has launched so far (for launch accounting).  Local. */
int mpxa_launch_count(mpxa_comm_t comm, uint64_t *count);

/* Collective registration of a device buffer for direct peer writes (multi-process mode;
 * a no-op in single-process mode): every process calls it with a buffer of its own; the
 * cudaMalloc allocation holding ptr becomes a window (its CUDA IPC handle is exchanged through
 * the bootstrap and opened by every peer), so later collectives into any buffer inside it
 * resolve peers' destinations on the device (window id + offset in the clear-to-send message).
 * The whole [ptr, ptr+bytes) range must lie in one cudaMalloc allocation, and that allocation
 * must stay allocated until mpxa_finalize: windows are never unmapped (mpxa_deregister is a
 * no-op), so an allocation freed and re-made at the same address (e.g. after
 * torch.cuda.empty_cache()) would still resolve to the peers' old mapping.  Persistent *_init
 * calls register their recvbuf implicitly.  Errors: MPXA_ERR_ARG (NULL, or ptr not inside a
 * device allocation), MPXA_ERR_NOMEM (more than 16 windows), MPXA_ERR_CUDA (IPC failure). */
int mpxa_register(mpxa_comm_t comm, void *ptr, size_t bytes);
int mpxa_deregister(mpxa_comm_t comm, void *ptr);   /* no-op (see mpxa_register) */

/* ---- one-shot collectives (MPI semantics) ---------------------------- */
/* count elements of dtype_size bytes per destination block. */
int mpxa_alltoall(const void *sendbuf, size_t count, size_t dtype_size, void *recvbuf,
                  mpxa_comm_t comm, mpxa_stream_t stream);
/* count elements of dtype_size bytes contributed by every rank. */
int mpxa_allgather(const void *sendbuf, size_t count, size_t dtype_size, void *recvbuf,
                   mpxa_comm_t comm, mpxa_stream_t stream);
/* R*p int64 counts/displacements in elements (host or device pointers; device arrays are
 * copied to the host synchronously). */
int mpxa_alltoallv(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                   size_t send_bytes_per_rank, void *recvbuf, const int64_t *recvcounts,
                   const int64_t *rdispls, size_t recv_bytes_per_rank, size_t dtype_size,
                   mpxa_comm_t comm, mpxa_stream_t stream);
/* Explicit-variant forms ("users can select a non-default algorithm"). */
int mpxa_alltoall_algo(const void *sendbuf, size_t count, size_t dtype_size, void *recvbuf,
                       mpxa_algo_t algo, mpxa_comm_t comm, mpxa_stream_t stream);
int mpxa_allgather_algo(const void *sendbuf, size_t count, size_t dtype_size, void *recvbuf,
                        mpxa_algo_t algo, mpxa_comm_t comm, mpxa_stream_t stream);
int mpxa_alltoallv_algo(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                        size_t send_bytes_per_rank, void *recvbuf, const int64_t *recvcounts,
                        const int64_t *rdispls, size_t recv_bytes_per_rank, size_t dtype_size,
                        mpxa_algo_t algo, mpxa_comm_t comm, mpxa_stream_t stream);

/* A2: counts exchange + displacement scan on the device (BASELINE.json cfg4 "counts/displs
 * exchanged then data").  d_sendcounts: DEVICE R*p int64; outputs DEVICE R*p int64:
 * d_recvcounts[t*p+j] = sendcounts of rank j for local rank t, d_rdispls = exclusive prefix
 * sum of each row.  One kernel; stream-ordered, no host synchronization. */
int mpxa_alltoallv_counts(const int64_t *d_sendcounts, int64_t *d_recvcounts,
                          int64_t *d_rdispls, mpxa_comm_t comm, mpxa_stream_t stream);

/* ---- Bruck step-level entry points (intermediate states) -------- */
/* Runs Bruck alltoall (rotation, then rounds 0..stop_stage-1) and writes T (rank-major,
 * p blocks of count*w per rank) to T_out.  stop_stage = 0 -> T after the local rotation;
 * stop_stage = k+1 -> after round k; stop_stage = -1 -> complete alltoall into T_out. */
int mpxa_alltoall_bruck_stage(const void *sendbuf, size_t count, size_t dtype_size,
                              void *T_out, int stop_stage, mpxa_comm_t comm,
                              mpxa_stream_t stream);
/* Same for Bruck allgather: T_r[0] = send_r, round k fills T[2^k, 2^k + n_k). */
int mpxa_allgather_bruck_stage(const void *sendbuf, size_t count, size_t dtype_size,
                               void *T_out, int stop_stage, mpxa_comm_t comm,
                               mpxa_stream_t stream);

/* ---- persistent forms (MPI-4 style) ------------- */
/* Buffers are bound at init and must stay allocated until mpxa_request_free.  `info` is
 * opaque and may be NULL. */
int mpxa_alltoall_init(const void *sendbuf, size_t count, size_t dtype_size, void *recvbuf,
                       mpxa_algo_t algo, mpxa_comm_t comm, const void *info,
                       mpxa_request_t *req);
int mpxa_allgather_init(const void *sendbuf, size_t count, size_t dtype_size, void *recvbuf,
                        mpxa_algo_t algo, mpxa_comm_t comm, const void *info,
                        mpxa_request_t *req);
int mpxa_alltoallv_init(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                        size_t send_bytes_per_rank, void *recvbuf, const int64_t *recvcounts,
                        const int64_t *rdispls, size_t recv_bytes_per_rank, size_t dtype_size,
                        mpxa_algo_t algo, mpxa_comm_t comm, const void *info,
                        mpxa_request_t *req);
int mpxa_start(mpxa_request_t req, mpxa_stream_t stream);  /* INACTIVE -> ACTIVE; enqueues   */
int mpxa_wait(mpxa_request_t req, mpxa_stream_t stream);   /* ACTIVE -> INACTIVE; enqueues the
                                                              device-side completion on
                                                              `stream` (no host round trip)  */
int mpxa_request_free(mpxa_request_t *req);
int mpxa_request_algorithm(mpxa_request_t req, mpxa_algo_t *algo);

/* ---- persistent neighborhood collectives (§2.2) ------ */
/* MPIX_Dist_graph_create_adjacent (Listing 4).  Collective over the comm's
 * processes.  Per local rank t (R of them, rank-major): indegree[t] in-neighbours listed in
 * `sources` (sum(indegree) entries, local rank 0's first), outdegree[t] out-neighbours in
 * `destinations`.  Repeated neighbours are separate edges, paired in order like MPI
 * messages (the j-th edge r->q with the j-th edge q<-r).  Weights may be NULL; they are stored
 * and, as the paper gives them no meaning, unused (SPEC.md decision).  `info` opaque, `reorder`
 * accepted and ignored.  The caller owns *topo (mpxa_topo_free); it references `comm`.
 * Errors: MPXA_ERR_ARG (NULL, negative degree, rank out of range).  Cross-process pairing is
 * checked at *_init. */
int mpxa_dist_graph_create_adjacent(mpxa_comm_t comm, const int *indegree, const int *sources,
                                    const int *sourceweights, const int *outdegree,
                                    const int *destinations, const int *destweights,
                                    const void *info, int reorder, mpxa_topo_t *topo);
int mpxa_topo_free(mpxa_topo_t *topo);

/* MPIX_Neighbor_alltoallv_init (Listing 4): out-edge k of local rank t sends
 * sendcounts[k] elements of dtype_size bytes from sendbuf + t*send_bytes_per_rank +
 * sdispls[k]*w; in-edge k receives recvcounts[k] elements at recvbuf + t*recv_bytes_per_rank
 * + rdispls[k]*w.  counts/displacements: host int64 arrays, one entry per edge, in the
 * topology's edge order (rank-major).  The whole schedule (one move per edge) is compiled and
 * uploaded here, once ("all setup costs ... incurred only once"); start/wait
 * then launch one kernel each.  Collective.  Errors: MPXA_ERR_ARG (bounds, overlap, dtype),
 * MPXA_ERR_MISMATCH (an edge without its partner, or partner counts differ). */
int mpxa_neighbor_alltoallv_init(const void *sendbuf, const int64_t *sendcounts,
                                 const int64_t *sdispls, size_t send_bytes_per_rank,
                                 void *recvbuf, const int64_t *recvcounts,
                                 const int64_t *rdispls, size_t recv_bytes_per_rank,
                                 size_t dtype_size, mpxa_topo_t topo, const void *info,
                                 mpxa_request_t *req);
/* Locality-aware variant ("unique indices for all values to be sent and
 * received ... eliminate a single value from being sent between a set of nodes multiple
 * times").  send_indices: one global index per sent element (edge by edge, in the order of
 * sendcounts); recv_indices: one per received element.  Equal indices must carry equal
 * values.  Ranks form groups of the comm's group_size (default: the ranks of one GPU); the
 * schedule forwards each group's unique (index) values for a remote group to the aggregator
 * leader_for, sends every unique index ONCE between the two groups, and fans
 * the values out to every (rank, offset) that needs them.  Extra error:
 * MPXA_ERR_TOPOLOGY when a received element's index differs from the one its edge sends. */
int mpxa_neighbor_alltoallv_locality_init(const void *sendbuf, const int64_t *sendcounts,
                                          const int64_t *sdispls, size_t send_bytes_per_rank,
                                          void *recvbuf, const int64_t *recvcounts,
                                          const int64_t *rdispls, size_t recv_bytes_per_rank,
                                          size_t dtype_size, const int64_t *send_indices,
                                          const int64_t *recv_indices, mpxa_topo_t topo,
                                          const void *info, mpxa_request_t *req);
/* One-shot MPI_Neighbor_alltoallv (Listing 3): the standard schedule,
 * compiled per call (the persistent form is the fast path). */
int mpxa_neighbor_alltoallv(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                            size_t send_bytes_per_rank, void *recvbuf, const int64_t *recvcounts,
                            const int64_t *rdispls, size_t recv_bytes_per_rank, size_t dtype_size,
                            mpxa_topo_t topo, mpxa_stream_t stream);

/* ---- partitioned point-to-point (§2.3) -------------- */
/* MPI-4 partitioned communication on the device: one match at initialization, per-partition
 * Pready from the host (stream-ordered) or from a producer kernel (include/mpxa_device.cuh),
 * Parrived as a host query or as a stream-ordered device wait.  No progress thread: each
 * readied partition is copied straight into the matched receiver's buffer by the GPU (peer
 * stores over NVLink when the receiver is on another GPU) and published with a per-partition
 * release flag tagged with the cycle number.
 *
 * psend_init: local rank `rank` (hosted by this process) will send `partitions` equal
 * partitions of `count` elements of dtype_size bytes from buf to rank `dest` with `tag`.
 * precv_init: local rank `rank` receives from `source` into buf, split into `partitions`
 * equal partitions (may differ from the sender's: "partitions of the same or different
 * sizes"; the total bytes must match).  Both return an unmatched request. */
int mpxa_psend_init(const void *buf, int partitions, size_t count, size_t dtype_size, int rank, int dest,
                    int tag, mpxa_comm_t comm, const void *info, mpxa_request_t *req);
int mpxa_precv_init(void *buf, int partitions, size_t count, size_t dtype_size, int rank, int source,
                    int tag, mpxa_comm_t comm, const void *info, mpxa_request_t *req);
/* The single match ("establishes a single match between a sender and receiver at
 * initialization"): collective over the comm's processes; pairs every unmatched send with the
 * first unmatched receive of the same (source, destination, tag), in creation order, maps the
 * receiver's buffer and flags for the sender, and readies both ends for mpxa_start.  Errors:
 * MPXA_ERR_MISMATCH (an unmatched end, or total bytes differ) -- no request is matched then. */
int mpxa_pmatch(mpxa_comm_t comm);
/* Mark sender partition(s) ready (Pready / Pready_range): enqueued on `stream` after the work
 * that produced them; the copy to the receiver starts when the stream reaches it ("early-bird
 * communication").  Request must be ACTIVE (after mpxa_start); each partition at
 * most once per cycle (else MPXA_ERR_ARG). */
int mpxa_pready(mpxa_request_t req, int partition, mpxa_stream_t stream);
int mpxa_pready_range(mpxa_request_t req, int partition_lo, int partition_hi, mpxa_stream_t stream);
/* Host query (Parrived): *flag = 1 iff receiver partition `partition` of the current cycle has
 * fully arrived (byte coverage by delivered sender partitions).  Non-blocking with respect to
 * the channel; reads the flags with a private stream. */
int mpxa_parrived(mpxa_request_t req, int partition, int *flag);
/* Device-side Parrived: work enqueued on `stream` after this call starts only once receiver
 * partitions [partition_lo, partition_hi) have arrived (consumers overlap the transfer). */
int mpxa_parrived_wait(mpxa_request_t req, int partition_lo, int partition_hi, mpxa_stream_t stream);
/* Device handle of an ACTIVE matched send request for mpxa_dev_pready (include/mpxa_device.cuh). */
int mpxa_psend_device(mpxa_request_t req, void *handle_out, size_t handle_bytes);
/* mpxa_start / mpxa_wait / mpxa_request_free apply: start begins a cycle on that end (the
 * receiver's start also clears the sender to write); wait enqueues, on `stream`, the wait for
 * every partition of the cycle (sender: delivered; receiver: arrived). */

/* ---- variant registry and selector --------------------- */
int mpxa_set_algorithm(mpxa_comm_t comm, mpxa_op_t op, mpxa_algo_t algo); /* DEFAULT = selector */
int mpxa_get_algorithm(mpxa_comm_t comm, mpxa_op_t op, size_t bytes, mpxa_algo_t *chosen);
int mpxa_list_algorithms(mpxa_op_t op, mpxa_algo_t *out, int *n);  /* *n in: capacity; out: count */
/* Load a selector table (text, '#' comments), lines
 *     "op p ranks_per_proc gpus group_size max_bytes algo"   (or "op p ranks_per_proc max_bytes
 *     algo": any GPU count and group size),
 * op in {alltoall, alltoallv, allgather}, algo in {pairwise, bruck, hier, ring}.  For a call
 * the first line matching (op, p, R, G, g) with bytes <= max_bytes wins; bytes is the block /
 * contribution size, for alltoallv the mean pair segment of the global count matrix.  The
 * default algorithm is: mpxa_set_algorithm override > table > built-in fallback rules
 * (pairwise; hierarchical allgather across GPUs with several ranks per GPU beyond the eager
 * range).  Replaces the comm's table; MPXA_ERR_ARG on an unreadable file or a bad line.
 * Tables shipped: selector_b200.txt next to libmpxa.so (measured by bench.py --write-selector),
 * loaded at mpxa_init unless $MPXA_SELECTOR names another. */
int mpxa_load_selector(mpxa_comm_t comm, const char *path);
/* 64-bit digest of everything that chooses a launch's protocol, path or grid on the host:
 * every tuning knob, the selector table, forced variants (MPXA_ALGO) and the
 * initial heap size.  mpxa_init compares it across processes before any CUDA call and fails
 * with MPXA_ERR_MISMATCH on a difference (a process running the eager protocol against one
 * running the direct protocol would otherwise stall until the watchdog fires).  Local call.
 * Note: mpxa_load_selector / mpxa_set_algorithm after init change it; they must be called
 * identically on every process. */
int mpxa_config_digest(mpxa_comm_t comm, uint64_t *digest);

const char *mpxa_error_string(int status);
const char *mpxa_algo_name(mpxa_algo_t algo);

#ifdef __cplusplus
}
#endif
#endif /* MPXA_H */

/*
 * mpxa_plan.h -- host-only introspection of the schedules libmpxa compiles (no CUDA calls,
 * usable on a machine without a GPU).  Tests use it to simulate a schedule on the CPU and
 * check its message counts against the closed forms of SURVEY.md §8(c) C.6.
 *
 * A plan is the per-GPU program one collective call runs: steps of moves (byte copies
 * between rank buffers) executed by the GPU that owns the source rank.
 *   op    : mpxa_op_t;  algo: mpxa_algo_t (not DEFAULT);  p = R * G ranks, R per GPU;
 *   g     : hierarchical group size (HIER only);
 *   stop_stage: -1 for the complete collective, else the Bruck stage entry-point truncation;
 *   c, sd, rd: ALLTOALLV only, full p x p int64 matrices (elements): c[s*p+j] sent by s to j,
 *              sd[s*p+j] its displacement in s's sendbuf, rd[j*p+s] the displacement in j's
 *              recvbuf of the segment from s.  Ignored (may be NULL) for uniform ops, whose
 *              units are whole blocks.
 * The handle is owned by the caller and released with mpxa_plan_free.
 */
#ifndef MPXA_PLAN_H
#define MPXA_PLAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t src_off, dst_off, len;   /* units                                   */
    uint32_t flow;                   /* identity of the data moved (origin block / segment) */
    uint16_t src_rank, dst_rank;
    uint8_t src_kind, dst_kind;      /* 0 send buffer, 1 recv buffer, 2 library workspace,
                                        3 eager staging (mpxa_plan_eager) */
    uint8_t fanout;                  /* 1: to every rank's dst_kind buffer at dst_off;
                                        2: to every rank of the executing GPU (eager plans) */
    uint8_t pad[5];
} mpxa_plan_move;

typedef struct {
    int32_t move_begin, move_end;    /* moves sorted by flow within the step     */
    uint32_t signal_mask, wait_mask; /* peer GPUs written / writing in this step */
    int64_t total_len, max_len;
    int32_t flow_index;              /* internal                                 */
    int32_t dense_base;              /* >= 0: move k carries flow dense_base + k */
} mpxa_plan_step;

typedef struct {
    int64_t nsteps, work_units, max_move, max_step_units, signals, total_moves, nflows, max_step_moves;
} mpxa_plan_info_t;

int mpxa_plan_build(int op, int algo, int p, int R, int G, int g, int stop_stage,
                    const int64_t *c, const int64_t *sd, const int64_t *rd, void **plan);
/* f1 neighbor alltoallv schedule from a GLOBAL graph (all p ranks, rank-major edge lists as
 * in mpxa_dist_graph_create_adjacent; counts/displacements per edge): locality = 0 standard,
 * 1 locality-aware with groups of g ranks and per-element global indices (else NULL).
 * Returns the mpxa status of the validation (MPXA_ERR_MISMATCH / _TOPOLOGY / _ARG). */
int mpxa_plan_build_neighbor(int p, int R, int G, int g, int locality, const int *indeg, const int *src,
                             const int64_t *rc, const int64_t *rd, const int *outdeg, const int *dst,
                             const int64_t *sc, const int64_t *sd, const int64_t *send_idx,
                             const int64_t *recv_idx, void **plan);
/* The eager (LL) form of a multi-GPU plan for `unit` bytes per unit -- what small launches
 * run (SURVEY.md §8 A9 "epoch-parity staging for eager mode"): a move whose destination is on
 * peer GPU d becomes a SEND move with dst_kind 3 (staging), dst_rank = d, dst_off = word
 * offset (4 payload bytes per 8-byte word, each word carrying the launch's flag) on the
 * source GPU, and a RECEIVE move with src_kind 3, src_rank = source GPU, src_off = word
 * offset on GPU d.  Fan-out moves keep fanout = 2 (this GPU's ranks only) plus one stream per
 * peer GPU.  In each step the receive moves come last; wait_mask = their number.  Pairs
 * without data exchange one flag word (len 0).  MPXA_ERR_ALGO when G < 2 or a GPU pair needs
 * more than 32768 words.  Released with mpxa_plan_free. */
int mpxa_plan_eager(const void *plan, size_t unit, void **eager);
int mpxa_plan_info(const void *plan, mpxa_plan_info_t *info);
/* copies GPU `gpu`'s steps / moves; *n in: capacity, out: count */
int mpxa_plan_steps(const void *plan, int gpu, mpxa_plan_step *out, int *n);
int mpxa_plan_moves(const void *plan, int gpu, mpxa_plan_move *out, int *n);
int mpxa_plan_free(void *plan);

#ifdef __cplusplus
}
#endif
#endif /* MPXA_PLAN_H */

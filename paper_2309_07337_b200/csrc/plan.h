// Schedule builders: compile one collective call into a per-GPU program of steps and moves
// (mpxa_internal.h).  Pure host logic, no CUDA calls -- exported for CPU tests through
// mpxa_plan_* in plan_api.cpp.
#pragma once
#include <stdint.h>

#include <unordered_map>
#include <vector>

#include "mpxa_internal.h"

namespace mpxa {

struct Program {
    int p = 0, R = 1, G = 1;
    std::vector<std::vector<Step>> steps;  // [G][nsteps]
    std::vector<std::vector<Move>> moves;  // [G][...]
    std::vector<std::vector<int32_t>> findex;  // [G][...] per-step flow indexes
    int nflows = 1;
    int64_t work_units = 0;                // WORK units needed per rank
    int64_t max_move = 0;                  // longest move (units)
    int64_t max_step_units = 0;            // max over (GPU, step) of the summed move units
    int64_t max_step_moves = 0;            // max over (GPU, step) of the move count
    int64_t signals = 0;                   // inter-GPU signals per launch (GPU-pair messages)
    int nsteps() const { return steps.empty() ? 0 : (int)steps[0].size(); }
};

enum Algo { A_DEFAULT = 0, A_PAIRWISE = 1, A_BRUCK = 2, A_HIER = 3, A_RING = 4, A_LOCALITY = 5 };

// Uniform ops: units are blocks (count * dtype_size bytes).
//   stop_stage: -1 complete; >= 0 truncated Bruck ending with a T dump into RECV.
// hier_staged: A_HIER with group = GPU (g == R) in its literal three-step form (gather to
// the leader, exchange, redistribute); by default that case compiles to the fused form.
bool build_alltoall(Program &P, int algo, int p, int R, int G, int g, int stop_stage, bool hier_staged = false);
bool build_allgather(Program &P, int algo, int p, int R, int G, int stop_stage, int g = 1);
// v-op: units are elements.  c, sd, rd are FULL p x p matrices:
//   c[s*p+j]  = elements rank s sends to j, sd[s*p+j] its displacement in s's sendbuf,
//   rd[j*p+s] = displacement in j's recvbuf of the segment from s.
bool build_alltoallv(Program &P, int algo, int p, int R, int G, int g, const int64_t *c,
                     const int64_t *sd, const int64_t *rd, bool hier_staged = false);

// f1 neighbor alltoallv.  Global graph, rank-major edge lists: indeg[p],
// src/rc/rd per in-edge; outdeg[p], dst/sc/sd per out-edge (elements).  Edges pair like MPI
// messages (j-th out-edge r->q with the j-th in-edge q<-r).  locality: groups of g
// consecutive ranks, send_idx / recv_idx = one global index per element, edge by edge.
// Returns 0, or an mpxa status (MPXA_ERR_ARG / _MISMATCH / _TOPOLOGY) without building.
int build_neighbor(Program &P, bool locality, int p, int R, int G, int g, const int *indeg, const int *src,
                   const int64_t *rc, const int64_t *rd, const int *outdeg, const int *dst, const int64_t *sc,
                   const int64_t *sd, const int64_t *send_idx, const int64_t *recv_idx, bool staged = false);

int ceil_log2(int p);

}  // namespace mpxa

// libmpxa: host-only schedule introspection (include/mpxa_plan.h) and test / debug hooks.
#include "runtime.h"

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
// sync, 32 owned flows, 64 WORK in shared memory, 128 warp-ring dynamic mode, 256 tiny kernel,
// 512 cooperative launch
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

// B1 -- the NCCL baseline of SURVEY.md §8(d) D.5 / BASELINE.md §4.1, in C++ so that no Python
// sits in the timed loop.  NOT part of the product: it is the "system library" MPI Advance
// layers over, measured on the same buffers and streams as mpxa.
//
//   alltoall(v): ncclGroupStart; for each peer ncclSend + ncclRecv of that pair's bytes
//                (ncclUint8); ncclGroupEnd
//   allgather:   ncclAllGather, and the grouped send/recv form
//
// Timing: warm-up calls, then `iters` calls back to back between CUDA events on the caller's
// stream (per-call device us), or -- for small messages -- `iters` calls captured in ONE
// CUDA graph, replayed 5 times, median.  The caller takes the max over
// ranks.  All entry points return 0 on success, else an ncclResult_t / cudaError_t code
// (>= 1000 for CUDA errors).
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

namespace {

int nck(ncclResult_t r) { return r == ncclSuccess ? 0 : (int)r; }
int cck(cudaError_t e) { return e == cudaSuccess ? 0 : 1000 + (int)e; }

#define TRY(x)               \
    do {                     \
        int rc_ = (x);       \
        if (rc_) return rc_; \
    } while (0)

struct B1 {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
};

// one collective call of `op` (B1_* below); bytes = block / contribution bytes, or the
// per-peer byte arrays for alltoallv
int one(B1 *b, int op, const char *send, char *recv, size_t bytes, const int64_t *sc, const int64_t *sd,
        const int64_t *rc, const int64_t *rd, cudaStream_t st) {
    const int n = b->nranks;
    switch (op) {
        case 0:   // alltoall: block j of send -> rank j; block j of recv <- rank j
            TRY(nck(ncclGroupStart()));
            for (int j = 0; j < n; j++) {
                TRY(nck(ncclSend(send + (size_t)j * bytes, bytes, ncclUint8, j, b->comm, st)));
                TRY(nck(ncclRecv(recv + (size_t)j * bytes, bytes, ncclUint8, j, b->comm, st)));
            }
            return nck(ncclGroupEnd());
        case 1:   // allgather (the collective)
            return nck(ncclAllGather(send, recv, bytes, ncclUint8, b->comm, st));
        case 2:   // allgather as grouped send/recv
            TRY(nck(ncclGroupStart()));
            for (int j = 0; j < n; j++) {
                TRY(nck(ncclSend(send, bytes, ncclUint8, j, b->comm, st)));
                TRY(nck(ncclRecv(recv + (size_t)j * bytes, bytes, ncclUint8, j, b->comm, st)));
            }
            return nck(ncclGroupEnd());
        case 3:   // alltoallv, counts / displacements in BYTES (host arrays of nranks)
            TRY(nck(ncclGroupStart()));
            for (int j = 0; j < n; j++) {
                if (sc[j]) TRY(nck(ncclSend(send + sd[j], (size_t)sc[j], ncclUint8, j, b->comm, st)));
                if (rc[j]) TRY(nck(ncclRecv(recv + rd[j], (size_t)rc[j], ncclUint8, j, b->comm, st)));
            }
            return nck(ncclGroupEnd());
        default:
            return (int)ncclInvalidArgument;
    }
}

}  // namespace

extern "C" {

int b1_version(int *v) { return nck(ncclGetVersion(v)); }

int b1_unique_id(void *out, size_t n) {
    if (n < sizeof(ncclUniqueId)) return (int)ncclInvalidArgument;
    ncclUniqueId id;
    TRY(nck(ncclGetUniqueId(&id)));
    memcpy(out, &id, sizeof id);
    return 0;
}

int b1_init(void **h, int nranks, int rank, const void *id, int device) {
    TRY(cck(cudaSetDevice(device)));
    B1 *b = new B1();
    b->nranks = nranks;
    b->rank = rank;
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    int rc = nck(ncclCommInitRank(&b->comm, nranks, u, rank));
    if (rc) { delete b; return rc; }
    *h = b;
    return 0;
}

int b1_finalize(void *h) {
    B1 *b = (B1 *)h;
    if (!b) return 0;
    int rc = nck(ncclCommDestroy(b->comm));
    delete b;
    return rc;
}

// one stream-ordered call (correctness checks)
int b1_call(void *h, int op, const void *send, void *recv, size_t bytes, const int64_t *sc, const int64_t *sd,
            const int64_t *rc, const int64_t *rd, void *stream) {
    return one((B1 *)h, op, (const char *)send, (char *)recv, bytes, sc, sd, rc, rd, (cudaStream_t)stream);
}

// device us per call: iters calls between events (graph = 0) or one graph of iters calls,
// median of 5 replays (graph = 1)
int b1_time(void *h, int op, const void *send, void *recv, size_t bytes, const int64_t *sc, const int64_t *sd,
            const int64_t *rc, const int64_t *rd, void *stream, int warmup, int iters, int graph, double *us) {
    B1 *b = (B1 *)h;
    cudaStream_t st = (cudaStream_t)stream;
    const char *s = (const char *)send;
    char *r = (char *)recv;
    for (int i = 0; i < warmup; i++) TRY(one(b, op, s, r, bytes, sc, sd, rc, rd, st));
    TRY(cck(cudaStreamSynchronize(st)));
    cudaEvent_t e0, e1;
    TRY(cck(cudaEventCreate(&e0)));
    TRY(cck(cudaEventCreate(&e1)));
    int rc2 = 0;
    if (!graph) {
        TRY(cck(cudaEventRecord(e0, st)));
        for (int i = 0; i < iters && !rc2; i++) rc2 = one(b, op, s, r, bytes, sc, sd, rc, rd, st);
        TRY(cck(cudaEventRecord(e1, st)));
        TRY(cck(cudaEventSynchronize(e1)));
        float ms = 0;
        TRY(cck(cudaEventElapsedTime(&ms, e0, e1)));
        *us = 1e3 * ms / iters;
    } else {
        // capture on a private non-blocking stream ordered after the caller's (the caller's
        // stream may be the legacy default stream, which cannot be captured)
        cudaStream_t cs;
        cudaEvent_t ord;
        TRY(cck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)));
        TRY(cck(cudaEventCreateWithFlags(&ord, cudaEventDisableTiming)));
        TRY(cck(cudaEventRecord(ord, st)));
        TRY(cck(cudaStreamWaitEvent(cs, ord, 0)));
        st = cs;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        TRY(cck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal)));
        for (int i = 0; i < iters && !rc2; i++) rc2 = one(b, op, s, r, bytes, sc, sd, rc, rd, st);
        TRY(cck(cudaStreamEndCapture(st, &g)));
        if (rc2) return rc2;
        TRY(cck(cudaGraphInstantiate(&ge, g, 0)));
        TRY(cck(cudaGraphLaunch(ge, st)));   // upload + warm
        TRY(cck(cudaStreamSynchronize(st)));
        std::vector<double> t;
        for (int k = 0; k < 5; k++) {
            TRY(cck(cudaEventRecord(e0, st)));
            TRY(cck(cudaGraphLaunch(ge, st)));
            TRY(cck(cudaEventRecord(e1, st)));
            TRY(cck(cudaEventSynchronize(e1)));
            float ms = 0;
            TRY(cck(cudaEventElapsedTime(&ms, e0, e1)));
            t.push_back(1e3 * ms / iters);
        }
        std::sort(t.begin(), t.end());
        *us = t[2];
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        TRY(cck(cudaEventRecord(ord, cs)));
        TRY(cck(cudaStreamWaitEvent((cudaStream_t)stream, ord, 0)));
        TRY(cck(cudaStreamSynchronize(cs)));
        cudaEventDestroy(ord);
        cudaStreamDestroy(cs);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return rc2;
}

}  // extern "C"

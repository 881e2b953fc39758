// libmpxa host runtime: argument checks (all before any data moves), the
// alltoall / allgather / alltoallv / neighbor implementations, persistent requests
// and their C ABI entry points.
#include "runtime.h"

namespace mpxa_rt {

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
                 mpxa_comm_t c, cudaStream_t stream, mpxa_request_t *req, int stage,
                 bool force_bruck) {
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


}  // namespace mpxa_rt

extern "C" {

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

}  // extern "C"

// libmpxa host runtime: MPI-4 partitioned point-to-point (§2.3).
#include "runtime.h"

extern "C" {

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

}  // extern "C"

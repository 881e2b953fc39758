// libmpxa host runtime: communicator bootstrap and IPC symmetric memory, tuning knobs and their
// cross-process digest, and the comm / registration entry points of the C ABI
// (MPIX_Comm_init analog: §2.1).
#include "runtime.h"

namespace mpxa_rt {

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
    if (const char *e = getenv("MPXA_NO_PREFETCH")) c->prefetch = atoi(e) ? 0 : 1;
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
    const int64_t v[] = {c->force_ns, c->force_nf, c->force_big, c->force_exec, c->pdl, c->dyn, c->wring, c->wslack, c->tiny, c->tiny_even, c->dyn_pieces, c->prefetch,
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

}  // namespace mpxa_rt

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

}  // extern "C"

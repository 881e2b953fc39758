// libmpxa host runtime: compiled programs (upload, per-unit companions, caches), CTA grid
// sizing and the launch decisions of every collective (which kernel, mode and grid).
#include "runtime.h"

namespace mpxa_rt {

void prog_facts(DevProg &dp) {
    const Program &P = dp.host;
    dp.max_gpu_moves = 0;
    dp.max_gpu_bytes_units = 0;
    dp.dyn_tiles = 0;
    for (int s = 0; s < P.nsteps(); s++) {
        int64_t mx = 0;
        for (int g = 0; g < P.G; g++) mx = std::max<int64_t>(mx, P.steps[g][s].move_end - P.steps[g][s].move_begin);
        dp.dyn_tiles += std::max<int64_t>(1, (mx + kMoveTile - 1) / kMoveTile);
    }
    dp.uniform_len = true;
    dp.fanout = false;
    for (const auto &mv : P.moves)
        for (const Move &m : mv) {
            if (m.len != P.max_move) dp.uniform_len = false;
            if (m.fanout) dp.fanout = true;
        }
    for (const auto &mv : P.moves) {
        dp.max_gpu_moves = std::max<int64_t>(dp.max_gpu_moves, (int64_t)mv.size());
        int64_t u = 0;
        for (const Move &m : mv) u += m.len;
        dp.max_gpu_bytes_units = std::max(dp.max_gpu_bytes_units, u);
    }
}

size_t serialize(const Program &P, std::vector<char> &buf, uintptr_t dbase) {
    const int G = P.G;
    size_t off = sizeof(GpuProg) * G;
    std::vector<size_t> soff(G), moff(G), foff(G);
    for (int g = 0; g < G; g++) { soff[g] = off; off += sizeof(Step) * P.steps[g].size(); }
    for (int g = 0; g < G; g++) { moff[g] = off; off += sizeof(Move) * P.moves[g].size(); }
    for (int g = 0; g < G; g++) { foff[g] = off; off += sizeof(int32_t) * P.findex[g].size(); }
    buf.assign(off, 0);
    for (int g = 0; g < G; g++) {
        GpuProg gp{};
        gp.steps = (const Step *)(dbase + soff[g]);
        gp.moves = (const Move *)(dbase + moff[g]);
        gp.findex = (const int32_t *)(dbase + foff[g]);
        gp.nsteps = (int32_t)P.steps[g].size();
        gp.nmoves = (int32_t)P.moves[g].size();
        memcpy(buf.data() + sizeof(GpuProg) * g, &gp, sizeof gp);
        if (!P.steps[g].empty()) memcpy(buf.data() + soff[g], P.steps[g].data(), sizeof(Step) * P.steps[g].size());
        if (!P.moves[g].empty()) memcpy(buf.data() + moff[g], P.moves[g].data(), sizeof(Move) * P.moves[g].size());
        if (!P.findex[g].empty())
            memcpy(buf.data() + foff[g], P.findex[g].data(), sizeof(int32_t) * P.findex[g].size());
    }
    return off;
}

size_t serialized_size(const Program &P) {
    size_t n = sizeof(GpuProg) * P.G;
    for (int g = 0; g < P.G; g++)
        n += sizeof(Step) * P.steps[g].size() + sizeof(Move) * P.moves[g].size() +
             sizeof(int32_t) * P.findex[g].size();
    return n;
}


int upload_program(const Program &P, std::shared_ptr<DevProg> &out) {
    auto dp = std::make_shared<DevProg>();
    size_t n = serialized_size(P);
    CK(cudaMalloc(&dp->dmem, n ? n : 16));
    std::vector<char> buf;
    serialize(P, buf, (uintptr_t)dp->dmem);
    int rc = h2d_complete(dp->dmem, buf.data(), n);
    if (rc) { cudaFree(dp->dmem); return rc; }
    dp->gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + P.G);
    dp->bytes = n;
    dp->host = P;
    dp->nsteps = P.nsteps();
    prog_facts(*dp);
    out = dp;
    return MPXA_SUCCESS;
}

// The variable-piece companion of dp: moves longer than chop units become chop-unit moves
// (same flow, order and kinds), so tiles of kSmallThreads moves carry comparable piece
// counts and no CTA inherits a tile of whole long moves.  Small kernel only (no findex).
int var_program(const DevProg &dp, int64_t chop, const DevProg *&out) {
    out = nullptr;
    auto have = dp.var.find(chop);
    if (have != dp.var.end()) { out = have->second.get(); return MPXA_SUCCESS; }
    if (dp.var.size() >= kMaxCompanions) return MPXA_SUCCESS;
    {
        const Program &P = dp.host;
        Program Q;
        Q.p = P.p; Q.R = P.R; Q.G = P.G;
        Q.nflows = P.nflows;
        Q.work_units = P.work_units;
        Q.max_step_units = P.max_step_units;
        Q.signals = P.signals;
        Q.max_move = std::min<int64_t>(P.max_move, chop);
        Q.steps.resize(P.G);
        Q.moves.resize(P.G);
        Q.findex.assign(P.G, {});
        for (int g = 0; g < P.G; g++)
            for (const Step &st0 : P.steps[g]) {
                Step st = st0;
                st.move_begin = (int32_t)Q.moves[g].size();
                for (int32_t i = st0.move_begin; i < st0.move_end; i++) {
                    const Move &m = P.moves[g][i];
                    int64_t o = 0;
                    do {
                        Move x = m;
                        x.src_off += o;
                        x.dst_off += o;
                        x.len = std::min<int64_t>(chop, m.len - o);
                        Q.moves[g].push_back(x);
                        o += chop;
                    } while (o < m.len);
                }
                st.move_end = (int32_t)Q.moves[g].size();
                st.max_len = std::min<int64_t>(st.max_len, chop);
                st.flow_index = 0;
                st.dense_base = -1;
                Q.max_step_moves = std::max<int64_t>(Q.max_step_moves, st.move_end - st.move_begin);
                Q.steps[g].push_back(st);
            }
        auto v = std::shared_ptr<DevProg>(new DevProg, [](DevProg *d) {
            if (d->dmem) cudaFree(d->dmem);
            delete d;
        });
        size_t n = serialized_size(Q);
        CK(cudaMalloc(&v->dmem, n ? n : 16));
        std::vector<char> buf;
        serialize(Q, buf, (uintptr_t)v->dmem);
        int rc = h2d_complete(v->dmem, buf.data(), n);
        if (rc) return rc;
        v->gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + Q.G);
        v->bytes = n;
        v->host = std::move(Q);
        v->nsteps = v->host.nsteps();
        prog_facts(*v);
        dp.var[chop] = v;
        out = v.get();
    }
    return MPXA_SUCCESS;
}

// Upload a companion program (small kernel only: no flow index) as a self-freeing DevProg.
static int upload_companion(Program &&Q, std::shared_ptr<DevProg> &out) {
    auto v = std::shared_ptr<DevProg>(new DevProg, [](DevProg *d) {
        if (d->dmem) cudaFree(d->dmem);
        delete d;
    });
    size_t n = serialized_size(Q);
    CK(cudaMalloc(&v->dmem, n ? n : 16));
    std::vector<char> buf;
    serialize(Q, buf, (uintptr_t)v->dmem);
    int rc = h2d_complete(v->dmem, buf.data(), n);
    if (rc) return rc;
    v->gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + Q.G);
    v->bytes = n;
    v->host = std::move(Q);
    v->nsteps = v->host.nsteps();
    prog_facts(*v);
    out = v;
    return MPXA_SUCCESS;
}

// Eager (LL) companion of a program for one unit ("epoch-parity staging for
// eager mode"): every move whose destination is on a peer GPU d becomes
//   on its GPU g:  a SEND move to (BK_LL, d, word offset w) -- the payload as 4-byte words,
//                  each stored with the launch's flag in one 8-byte word into d's staging;
//   on GPU d:      a RECEIVE move (BK_LL, g, w) -> the original destination, which polls
//                  the words until they carry the flag.
// Fan-out moves (allgather direct) keep a local fan-out (fanout = 2: this GPU's ranks) and
// send one stream per peer GPU, which the peer fans out to its own ranks.  Word offsets run
// per (g, d) pair across all steps of the launch; a pair without data still exchanges one
// flag word, so every GPU hears from every peer in every eager launch -- which is what makes
// the two staging parities safe to alternate.  In each step the receive moves come last
// (Step::wait_mask = their number): a CTA issues all its sends before it polls.
// Returns false when a pair needs more than kLLWords words or a GPU more moves than the
// small kernel caches.
bool build_ll(const Program &P, uint64_t unit, int R, Program &Q, int64_t max_words) {
    const int G = P.G, ns = P.nsteps();
    Q = Program();
    Q.p = P.p; Q.R = P.R; Q.G = G;
    Q.nflows = P.nflows;
    Q.work_units = P.work_units;
    Q.max_step_units = P.max_step_units;
    Q.max_move = P.max_move;
    Q.signals = 0;
    Q.steps.assign(G, {});
    Q.moves.assign(G, {});
    Q.findex.assign(G, {});
    std::vector<int64_t> wc((size_t)G * G, 0);
    auto words = [&](const Move &m) { return std::max<int64_t>(1, (int64_t)((m.len * unit + 3) / 4)); };
    for (int s = 0; s < ns; s++) {
        std::vector<std::vector<Move>> out(G), in(G);
        for (int g = 0; g < G; g++) {
            const Step &st = P.steps[g][s];
            for (int32_t i = st.move_begin; i < st.move_end; i++) {
                const Move &m = P.moves[g][i];
                if (m.fanout) {
                    Move x = m;
                    x.fanout = 2;
                    out[g].push_back(x);
                }
                for (int d = 0; d < G; d++) {
                    if (d == g) continue;
                    if (!m.fanout && (int)m.dst_rank / R != d) continue;
                    int64_t &w0 = wc[(size_t)g * G + d];
                    w0 += w0 & 1;   // even word offsets: 16-byte aligned pairs of words
                    Move snd = m, rcv = m;
                    snd.fanout = 0;
                    snd.dst_kind = BK_LL;
                    snd.dst_rank = (uint16_t)d;
                    snd.dst_off = wc[(size_t)g * G + d];
                    rcv.fanout = m.fanout ? 2 : 0;
                    rcv.src_kind = BK_LL;
                    rcv.src_rank = (uint16_t)g;
                    rcv.src_off = wc[(size_t)g * G + d];
                    wc[(size_t)g * G + d] += words(m);
                    out[g].push_back(snd);
                    in[d].push_back(rcv);
                }
                if (!m.fanout && (int)m.dst_rank / R == g) out[g].push_back(m);
            }
        }
        if (s == 0)   // flag-only words for pairs without data in the whole launch
            for (int g = 0; g < G; g++)
                for (int d = 0; d < G; d++) {
                    if (d == g) continue;
                    bool any = false;
                    for (int s2 = 0; s2 < ns && !any; s2++) {
                        const Step &st = P.steps[g][s2];
                        for (int32_t i = st.move_begin; i < st.move_end && !any; i++) {
                            const Move &m = P.moves[g][i];
                            any = m.fanout || (int)m.dst_rank / R == d;
                        }
                    }
                    if (any) continue;
                    Move snd{}, rcv{};
                    snd.src_kind = BK_SEND;
                    snd.src_rank = (uint16_t)(g * R);
                    snd.dst_kind = BK_LL;
                    snd.dst_rank = (uint16_t)d;
                    rcv.src_kind = BK_LL;
                    rcv.src_rank = (uint16_t)g;
                    rcv.dst_kind = BK_RECV;
                    rcv.dst_rank = (uint16_t)(d * R);
                    wc[(size_t)g * G + d] = 1;
                    out[g].push_back(snd);
                    in[d].push_back(rcv);
                }
        for (int g = 0; g < G; g++) {
            Step st = P.steps[g][s];
            st.move_begin = (int32_t)Q.moves[g].size();
            for (const Move &m : out[g]) Q.moves[g].push_back(m);
            for (const Move &m : in[g]) Q.moves[g].push_back(m);
            st.move_end = (int32_t)Q.moves[g].size();
            st.signal_mask = 0;
            st.wait_mask = (uint32_t)in[g].size();
            st.flow_index = 0;
            st.dense_base = -1;
            Q.max_step_moves = std::max<int64_t>(Q.max_step_moves, st.move_end - st.move_begin);
            Q.steps[g].push_back(st);
        }
    }
    for (int64_t w : wc)
        if (w > std::min<int64_t>(max_words, kLLWords)) return false;
    for (int g = 0; g < G; g++)
        if (Q.moves[g].size() > (size_t)kSmallMovesSmem) return false;
    return true;
}

// The eager companion of dp for `unit`, built on first use (never inside a stream capture:
// the upload is synchronous).  nullptr when ineligible or not available.
static const DevProg *ll_program(mpxa_comm_t c, const DevProg &dp, uint64_t unit, cudaStream_t stream) {
    auto have = dp.ll.find(unit);
    if (have != dp.ll.end()) return have->second.get();
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (dp.per_call || cudaStreamIsCapturing(stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return nullptr;
    if (dp.ll.size() >= kMaxCompanions) return nullptr;
    std::shared_ptr<DevProg> &slot = dp.ll[unit];   // null = ineligible (kept: decided once)
    Program Q;
    // measured (4 emulated GPUs, p = 4 / 8): eager wins up to the full 128 KiB staging per
    // GPU pair for single-step launches (pairwise alltoall 64 KiB pairs 16.0 -> 10.2 us; the
    // direct protocol's CTS + two system-scope releases cost more than eager's 2x bytes);
    // multi-step ones pay the 2x bytes and word stores in every step; re-measured after the
    // executor's per-GPU signalling: eager still wins at 64 KiB per pair (ring allgather 4 KiB
    // blocks 37.5 -> 19.7 us, Bruck alltoall 2 KiB 24.5 -> 16.2 us on 4 emulated GPUs)
    const int64_t max_words = (dp.nsteps > 1 ? c->ll_max_ms : c->ll_max) / 4;
    if (!build_ll(dp.host, unit, c->Rg, Q, max_words)) return nullptr;
    std::shared_ptr<DevProg> up;
    if (upload_companion(std::move(Q), up) != MPXA_SUCCESS) return nullptr;
    slot = up;
    return slot.get();
}

// Persistent *_init: build the eager companion now (collective, outside any stream capture),
// so a first start() inside a CUDA-graph capture already runs eager, the same in every process.
void prebuild_companions(mpxa_comm_t c, const DevProg &dp, uint64_t unit) {
    if (c->ll && c->G > 1 && c->p <= kRankTable) (void)ll_program(c, dp, unit, (cudaStream_t)0);
}

int cached_uniform(mpxa_comm_t c, int op, int algo, int stage, std::shared_ptr<DevProg> &out) {
    auto key = std::make_tuple(op, algo, stage, c->g);
    auto it = c->cache.find(key);
    if (it != c->cache.end()) { out = it->second; return MPXA_SUCCESS; }
    Program P;
    bool ok = op == MPXA_OP_ALLTOALL ? build_alltoall(P, algo, c->p, c->Rg, c->G, c->g, stage, c->hier_staged)
                                     : build_allgather(P, algo, c->p, c->Rg, c->G, stage, c->g);
    if (!ok) return MPXA_ERR_ALGO;
    int rc = upload_program(P, out);
    if (rc) return rc;
    c->cache[key] = out;
    return MPXA_SUCCESS;
}


uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

Grid choose_grid(mpxa_comm_t c, const Program &P, uint64_t unit) {
    const uint64_t L = (uint64_t)P.max_move * unit;          // longest move
    const uint64_t T = (uint64_t)P.max_step_units * unit;    // busiest step of one GPU
    Grid gr;
    // large steps stream through fewer, fatter pipelines; the rest through more CTAs
    gr.big = c->force_big >= 0 ? c->force_big > 0 : T / (uint64_t)c->cap_big >= kBigPerCta;
    const uint64_t cap = (uint64_t)(gr.big ? c->cap_big : c->cap_ctas);
    uint64_t nS = std::min<uint64_t>(cap, std::max<uint64_t>(1, cdiv(L, kSliceBytes)));
    uint64_t nF_bw = cdiv(T, nS * kBytesPerCta);              // enough CTAs for bandwidth
    uint64_t nF_lat = cdiv((uint64_t)P.max_step_moves, kMovesPerCta);  // ~1 move per LSU warp
    uint64_t nF = std::max<uint64_t>(1, std::max(nF_bw, nF_lat));
    nF = std::min<uint64_t>(nF, std::max<uint64_t>(1, cap / nS));
    nF = std::min<uint64_t>(nF, (uint64_t)P.nflows);
    if (c->force_ns > 0) nS = (uint64_t)c->force_ns;
    if (c->force_nf > 0) nF = std::min<uint64_t>((uint64_t)c->force_nf, (uint64_t)P.nflows);
    while (nS * nF > (uint64_t)kMaxCtas || nS * nF > cap) {
        if (nF > 1) nF--;
        else nS--;
    }
    // fill the machine: widen the slices' count to use every resident CTA slot when the
    // slices stay >= kMinSlice bytes
    if (c->force_ns <= 0 && nF >= 1) {
        uint64_t wide = cap / nF;
        if (wide > nS && L / wide >= kMinSlice) nS = wide;
        else if (wide > nS && L / kMinSlice > nS) nS = std::min<uint64_t>(wide, L / kMinSlice);
    }
    gr.nS = (int)std::max<uint64_t>(1, nS);
    gr.nF = (int)std::max<uint64_t>(1, nF);
    return gr;
}

// Fill launch parameters for a program on this comm.
int make_params(mpxa_comm_t c, ExecParams &E, const DevProg &dp, const char *send, char *recv,
                uint64_t unit, uint64_t send_stride, uint64_t recv_stride) {
    memset(&E, 0, sizeof E);
    E.progs = (const GpuProg *)dp.dmem;
    if (!c->emulated) E.prog = dp.gp[c->nprocs > 1 ? c->proc : 0];
    E.dc = c->dc;
    E.send = send;
    E.recv = recv;
    E.unit = unit;
    E.send_stride = send_stride;
    E.recv_stride = recv_stride;
    E.work_stride = (uint64_t)dp.host.work_units * unit;
    E.err = c->err_dev;
    E.timeout_ns = (int64_t)(c->timeout_s * 1e9);
    E.G = c->G;
    E.R = c->Rg;
    E.p = c->p;
    E.nflows = dp.host.nflows;
    E.my_gpu = c->emulated ? -1 : (c->nprocs > 1 ? c->proc : 0);
    E.mode = c->emulated ? 1 : (c->nprocs > 1 ? 2 : 0);
    // step 0 dense on EVERY GPU with one base flow and count (single program per launch
    // in modes 0 / 2; emulated launches need them equal across the virtual GPUs)
    E.d0_base = -1;
    if (dp.nsteps > 0) {
        const int g0 = c->emulated ? 0 : (c->nprocs > 1 ? c->proc : 0);
        const Step &s0 = dp.host.steps[g0][0];
        bool ok = s0.dense_base >= 0;
        if (c->emulated)
            for (int g = 1; g < c->G && ok; g++) {
                const Step &o = dp.host.steps[g][0];
                ok = o.dense_base == s0.dense_base && o.move_end == s0.move_end;
            }
        if (ok) { E.d0_base = s0.dense_base; E.d0_n = s0.move_end - s0.move_begin; }
    }
    if (c->nprocs > 1) {
        // remote recv bases are resolved on the device from the CTS message (window + offset)
        uintptr_t r = (uintptr_t)recv;
        int wi = -1;
        for (size_t w = 0; w < c->windows.size(); w++)
            if (r >= c->windows[w].base && r < c->windows[w].base + c->windows[w].size) { wi = (int)w; break; }
        if (wi < 0) return MPXA_ERR_UNREGISTERED;
        E.recv_win = (uint64_t)wi;
        E.recv_off = r - c->windows[wi].base;
    }
    return MPXA_SUCCESS;
}

// Cooperative level of a launch (kern_common.cuh launch_kernel): CTAs that wait on one another must
// be co-resident.  Emulated GPUs: cooperative (their CTA rows exchange flags; launches as in
// round 1, no PDL).  Across processes every CTA may wait on a peer GPU's CTAs, which wait on
// this grid's: cooperative + PDL, so no CTA spins while another of its grid is not scheduled
// (another stream's kernel holding SMs).  One GPU: only launches with per-step row barriers
// (barriers: several steps over several CTAs, not owned-flow).
static int coop_level(mpxa_comm_t c, bool barriers) {
    if (c->emulated) return 1;
    return (c->nprocs > 1 || barriers) ? 2 : 0;
}

// pdl: the launch may overlap the previous kernel's tail (the kernel waits on
// griddepcontrol before touching anything that kernel wrote).  Off for per-call programs,
// whose tables arrive by a cudaMemcpyAsync right before the launch.
int run_program(mpxa_comm_t c, const DevProg &dp, const char *send, char *recv, uint64_t unit,
                uint64_t send_stride, uint64_t recv_stride, cudaStream_t stream, const Grid *grid,
                bool pdl) {
    if (c->poisoned) return MPXA_ERR_TIMEOUT;
    if (dp.nsteps == 0) return MPXA_SUCCESS;
    size_t need = (size_t)dp.host.work_units * unit * c->Rg;
    int rc = ensure_work(c, need);
    if (rc) return rc;
    ExecParams E;
    rc = make_params(c, E, dp, send, recv, unit, send_stride, recv_stride);
    if (rc) return rc;
    const Grid gr = grid ? *grid : choose_grid(c, dp.host, unit);
    E.nS = gr.nS;
    E.nF = gr.nF;
    const TmaConfig tc = gr.big ? kTmaBig : kTmaMid;
    E.stages = tc.stages;
    E.chunk = tc.chunk;
    E.ahead = tc.ahead;
    ++c->epoch;   // host mirror only; the kernels keep the authoritative epoch in DevComm
    cudaError_t e;
    int coop = 0;   // cooperative level of the launch (coop_level)
    bool tiny = false;
    const uint64_t maxmove = (uint64_t)dp.host.max_move * unit;
    uint64_t ppm = 1;   // 16-B pieces per move, rounded up to a power of two (shift decode)
    while (ppm * 16 < maxmove) ppm <<= 1;
    // pieces per step, fan-out stores counted per destination (max_step_units counts them)
    const uint64_t slots = std::max<uint64_t>((uint64_t)dp.host.max_step_moves,
                                              (uint64_t)dp.host.max_step_units / std::max<int64_t>(1, dp.host.max_move)) * ppm;
    // moves of very different lengths (e.g. element runs next to whole blocks): max-move slots
    // per move are mostly empty -- the small kernel then counts pieces exactly per tile of moves
    const uint64_t exact = (uint64_t)dp.host.max_step_units * unit / 16 + (uint64_t)dp.host.max_step_moves;
    const bool var = !dp.uniform_len && exact * 4 < slots;
    const uint64_t items = var ? exact : slots;
    const bool one_step = dp.nsteps == 1;
    // Small-message kernel: multi-step programs with short moves and a step small enough for
    // one CTA; single-step programs (any number of CTAs) up to 2 MiB moves and 32 MiB of
    // source data per GPU -- measured on one B200: its LSU pieces beat the TMA executor's
    // fixed costs there (alltoall 64 KiB blocks 5.3 -> 3.8 us, allgather 1 MiB 17.9 -> 13.8 us,
    // alltoallv cfg4 64 KiB mean 9.2 -> 5.2 us); beyond, the executor streams better.
    const uint64_t src_vol = (uint64_t)dp.max_gpu_bytes_units * unit;
    // multi-step programs too large for one CTA but small in volume: several CTAs with a
    // barrier between steps (sync mode)
    const uint64_t step_vol = (uint64_t)dp.host.max_step_units * unit;
    // (measured: it wins where the static executor is poorly balanced -- uneven moves, or few
    // flows to spread over CTAs as in the allgathers; uniform alltoalls keep the barrier-free
    // static executor)
    const uint64_t per_cta = dp.fanout ? std::max<uint64_t>(32, c->small_items / 2) : c->small_items;
    const uint64_t n_own = std::max<uint64_t>(1, std::min<uint64_t>(std::min<uint64_t>(cdiv(items, per_cta),
                                                                                          (uint64_t)dp.host.nflows),
                                                                     (uint64_t)c->cap_small));
    const uint64_t own_vol = c->own_vol ? c->own_vol : c->emulated ? kSmallOwnVolEmu : kSmallOwnVol;
    const uint64_t own_per_cta = c->own_per_cta ? c->own_per_cta : c->emulated ? kSmallOwnPerCtaEmu : kSmallOwnPerCta;
    const bool own_ok = dp.uniform_len && step_vol <= own_vol && step_vol / n_own <= own_per_cta;
    const bool small_sync = !one_step && items > c->one_cta_items && maxmove <= kSmallSyncMove &&
                            step_vol <= kSmallSyncVol && c->small_sync &&
                            (!own_ok || dp.max_gpu_moves > kSmallMovesSmem) &&
                            (!dp.uniform_len || dp.host.nflows < 32 || dp.max_gpu_moves > kSmallMovesSmem);
    // uniform multi-step programs (flows of equal size, moved whole in every step): several
    // CTAs, each owning the flows f % nC == c through all steps -- no barrier needed
    // (measured, p=8: Bruck alltoall 4 KiB 13.9 -> 10.8 us, hier 9.8 -> 8.6 us at 16 KiB; from
    // 64 KiB blocks the TMA executor is faster again)
    const bool small_own = !one_step && !small_sync && items > c->one_cta_items && maxmove <= kSmallSyncMove &&
                           own_ok && c->small_sync && dp.max_gpu_moves <= kSmallMovesSmem;
    // (emulated GPUs share the SMs: a virtual GPU's small-kernel row has 1/G of them, and its
    // LSU pieces lose to the executor's TMA on long moves sooner -- measured: f1 halo, 2 MiB
    // moves on 4 emulated GPUs, 47 -> 32 us with the executor; cfg5's 64-256 KiB moves stay
    // 3x faster in the small kernel)
    const uint64_t max1 = c->emulated ? std::min<uint64_t>(c->small_max1, 1u << 20) : c->small_max1;
    const bool small = !c->force_exec &&
                       (one_step ? (maxmove <= max1 && src_vol <= c->small_vol1)
                                 : ((maxmove <= kSmallKernelMax && items <= c->one_cta_items) || small_sync ||
                                    small_own));
    if (small) {
        E.nS = E.nF = 1;
        E.small_a16 = unit % 16 == 0 && (uintptr_t)send % 16 == 0 && (uintptr_t)recv % 16 == 0 &&
                      send_stride % 16 == 0 && recv_stride % 16 == 0 && E.work_stride % 16 == 0;
        // int64 / double payloads: 8-byte words instead of 4-byte words and funnel shifts (eager
        // launches keep their own 4-byte word streams; a per-process choice -- no protocol
        // consequence across processes)
        E.small_a8 = !E.small_a16 && unit % 8 == 0 && (uintptr_t)send % 8 == 0 && (uintptr_t)recv % 8 == 0 &&
                     send_stride % 8 == 0 && recv_stride % 8 == 0 && E.work_stride % 8 == 0;
        E.small_a4 = !E.small_a16 && !E.small_a8 && unit % 4 == 0 && (uintptr_t)send % 4 == 0 &&
                     (uintptr_t)recv % 4 == 0 && send_stride % 4 == 0 && recv_stride % 4 == 0 &&
                     E.work_stride % 4 == 0;
        E.small_ppm = (int32_t)ppm;
        const DevProg *sp = &dp;
        // variable pieces: long moves split (companion program) unless the tables are per-call
        // or the stream is being captured (the companion's upload is synchronous)
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        const int64_t chop = std::max<int64_t>(1, c->var_chop / (int64_t)unit);
        if (var && !dp.per_call && c->var_chop > 0 && (uint64_t)dp.host.max_move * unit > (uint64_t)c->var_chop &&
            (dp.var.count(chop) ||
             (cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone))) {
            const DevProg *vp = nullptr;
            rc = var_program(dp, chop, vp);
            if (rc) return rc;
            if (vp) {
                sp = vp;
                E.progs = (const GpuProg *)sp->dmem;
                if (!c->emulated) E.prog = sp->gp[c->nprocs > 1 ? c->proc : 0];
            }
        }
        // eager (LL) mode: several GPUs, small launches -- the payload travels with its flags,
        // no CTS, no system-scope release (build_ll)
        if (c->ll && c->G > 1 && !var && c->p <= kRankTable) {
            if (const DevProg *lp = ll_program(c, dp, unit, stream)) {
                sp = lp;
                E.small_ll = 1;
                E.progs = (const GpuProg *)sp->dmem;
                if (!c->emulated) E.prog = sp->gp[c->nprocs > 1 ? c->proc : 0];
            }
        }
        size_t nmoves_g = 0;
        for (const auto &mv : sp->host.moves) nmoves_g = std::max(nmoves_g, mv.size());
        E.small_cache = nmoves_g <= (size_t)kSmallMovesSmem ? (int32_t)nmoves_g : 0;
        int nC = (one_step || small_sync || small_own)
                     ? (int)std::min<uint64_t>(cdiv(items, per_cta), (uint64_t)c->cap_small) : 1;
        if (small_own) nC = std::min<int>(nC, dp.host.nflows);
        E.dyn_sync = small_sync && nC > 1;
        E.small_own = small_own && nC > 1 ? nC : 0;
        if (E.small_ll && E.small_own) {   // eager steps take every piece of the step (no flow
            E.small_own = 0;               // ownership): CTAs meet at the row barrier instead
            E.dyn_sync = 1;
        }
        E.small_var = var && !E.small_own;
        if (E.small_var) {   // warp tiles of 32 moves, about var_tiles per CTA
            nC = (int)std::min<uint64_t>((uint64_t)c->cap_small,
                                         std::max<uint64_t>(1, cdiv(cdiv((uint64_t)sp->host.max_step_moves, 32),
                                                                    (uint64_t)c->var_tiles)));
            E.dyn_sync = !one_step && nC > 1;
        }
        // one CTA on one GPU, several steps, moves cached: the WORK rows live in the CTA's
        // shared memory (the kernel resolves WORK pointers there)
        const uint64_t wbytes = (uint64_t)dp.host.work_units * unit * (uint64_t)c->Rg;
        if (c->swork && !E.small_var && !E.small_own && nC <= 1 && c->G == 1 && !c->emulated && c->nprocs == 1 &&
            dp.nsteps > 1 && E.small_cache > 0 && c->p <= kRankTable && wbytes > 0 &&
            wbytes <= (uint64_t)kSmallWorkSmem)
            E.small_swork = 1;
        // few pieces per CTA and step: the smallest block (from small_nt = 64 threads) with one
        // piece per thread -- fewer idle warps contend for issue slots at every step (measured:
        // 4-5 % at <= 64 B; four pieces per thread in a smaller block lose up to 30 %)
        if (!E.small_var) {
            const uint64_t per_cta = cdiv(items, (uint64_t)std::max(1, nC));
            uint64_t nt = (uint64_t)c->small_nt;
            while (nt < 512 && (nt < per_cta || nt < (uint64_t)c->p || nt < (uint64_t)dp.nsteps)) nt *= 2;
            if (nt < 512) E.small_threads = (int32_t)nt;
        }
        // one step on one GPU, every move cached: the tiny kernel (no flags,
        // steps or rank tables -- the shortest instruction stream for a cold SM)
        tiny = c->tiny && one_step && c->G == 1 && !c->emulated && c->nprocs == 1 && !E.small_var &&
               !E.small_own && !E.small_ll && E.small_cache > 0 && sp == &dp;
        // several steps, one CTA, one GPU, every move cached: the tiny multi-step kernel
        const bool tiny_ms = c->tiny && !one_step && c->G == 1 && !c->emulated && c->nprocs == 1 &&
                             (nC <= 1 || E.small_own > 1) && !E.small_var && !E.dyn_sync && !E.small_ll &&
                             E.small_cache > 0 && dp.nsteps <= kMaxStepsSmem && sp == &dp;
        // one-step eager launches across GPUs: the tiny eager kernel (same word protocol)
        const bool tiny_ll = c->tiny && one_step && E.small_ll && !E.small_var && !E.small_own && E.small_cache > 0;
        if (tiny && c->tiny_even) {
            // the tiny kernel hands each CTA blockDim consecutive pieces: size the block to the
            // pieces the kernel decodes (fan-out: one per source piece, not per destination) over
            // the grid, a multiple of a warp, so every CTA of the grid gets work (measured, p = 8:
            // allgather 16 / 32 / 64 / 128 KiB 2.12 / 2.12 / 2.22 / 2.78 -> 1.50 / 1.55 / 1.59 /
            // 2.27 us -- the power-of-two block sized by fan-out-weighted pieces left 7 of 8 CTAs
            // idle; alltoall 16 KiB 1.52 -> 1.48)
            const uint64_t kitems = (uint64_t)dp.host.max_step_moves * ppm;
            const uint64_t nt = std::max<uint64_t>(64, std::min<uint64_t>(512, (cdiv(kitems, (uint64_t)std::max(1, nC)) + 31) / 32 * 32));
            E.small_threads = (int32_t)nt;
        }
        if (tiny) e = launch_tiny(E, std::max(1, nC), pdl && c->pdl, stream);
        else if (tiny_ms) {
            E.small_swork = 0;   // (the tiny multi-step kernel keeps WORK in global memory / L2)
            E.tiny_step_items = (int32_t)std::min<uint64_t>(INT32_MAX, (uint64_t)dp.host.max_step_moves * ppm);
            e = launch_tiny_ms(E, std::max(1, nC), pdl && c->pdl, stream);
        }
        else if (tiny_ll) {
            if (c->tiny_even) {   // (the same sizing: the pieces of the busiest GPU's eager program)
                const uint64_t kitems = (uint64_t)nmoves_g * ppm;
                E.small_threads = (int32_t)std::max<uint64_t>(
                    64, std::min<uint64_t>(512, (cdiv(kitems, (uint64_t)std::max(1, nC)) + 31) / 32 * 32));
            }
            coop = coop_level(c, !one_step && nC > 1 && !E.small_own);
            e = launch_tiny_ll(E, std::max(1, nC), c->emulated ? c->G : 1, coop, pdl && c->pdl, stream);
        } else {
            coop = coop_level(c, !one_step && nC > 1 && !E.small_own);
            e = launch_small(E, std::max(1, nC), c->emulated ? c->G : 1, coop, pdl && c->pdl, stream);
        }
        tiny = tiny || tiny_ll || tiny_ms;
    } else {
        int nC = gr.n();
        // dynamic mode: one step whose moves all fit the CTA's shared-memory move tile and
        // whose busiest GPU moves enough bytes for the tail of static slices to matter
        const int64_t ntiles = (dp.max_gpu_moves + kMoveTile - 1) / kMoveTile;
        if (c->dyn && dp.nsteps == 1 && ntiles <= kMaxDynTiles && dp.max_gpu_bytes_units > 0) {
            const uint64_t total = (uint64_t)dp.max_gpu_bytes_units * unit;
            const uint64_t avg = total / (uint64_t)std::max<int64_t>(1, dp.max_gpu_moves);
            // measured (p = 8..32 on one B200): the queues win once moves are large; with many
            // mid-size moves the per-tile setup costs more than the tail it removes
            if ((total >= c->dyn_min_total && avg >= kDynMinAvg) || (total >= kDynBigTotal && avg >= kDynMinMove)) {
                // the mid TMA ring at 2 CTAs / SM: twice the producers and LSU warps of the
                // big ring (the LSU queue needs the warps; the TMA queue is indifferent).  The
                // grid depends on the program only, so processes pair CTA flag slots 1:1.
                const TmaConfig tm = c->force_big > 0 ? kTmaBig : kTmaMid;
                E.stages = tm.stages;
                E.chunk = tm.chunk;
                E.ahead = tm.ahead;
                nC = c->force_big > 0 ? c->cap_big : c->cap_ctas;
                uint64_t U = total / ((uint64_t)nC * (uint64_t)c->dyn_pieces);
                U = std::max<uint64_t>((uint64_t)E.chunk, std::min<uint64_t>(U, kDynMaxPiece));
                // many move tiles (p >= 23 ranks on one GPU): each tile is classified by the whole
                // CTA while the producer stops issuing, so fewer, longer pieces pay (measured,
                // p = 32, 256 KiB blocks: 16 -> 48 KiB pieces, 93.2 -> 85.7 us; one or two
                // tiles: unchanged or slower)
                if (ntiles >= 4) U = std::max<uint64_t>(U, 3 * (uint64_t)E.chunk);
                U = U / (uint64_t)E.chunk * (uint64_t)E.chunk;
                // moves without fan-out (alltoall, alltoallv): pieces of at least two ring chunks
                // (measured, p = 8: alltoall 1 / 4 MiB blocks 22.3 / 82.5 -> 21.1 / 82.1 us;
                // fan-out pieces stay 16 KiB -- 32 KiB cost allgather 2-7 %)
                if (!dp.fanout) U = std::max<uint64_t>(U, 2 * (uint64_t)E.chunk);
                E.nS = nC;
                E.nF = 1;
                E.dyn_units = (int32_t)std::max<int64_t>(1, ntiles);
                E.dyn_u = (int32_t)U;
            }
        } else if (c->dyn && dp.nsteps > 1 && dp.dyn_tiles <= kMaxDynTiles &&
                   (c->force_sync > 0 || (dp.host.max_step_moves >= kDynSyncMoves && (uint64_t)dp.host.max_step_units * unit >= kDynSyncMin) ||
                    // moves of different lengths: static flow groups get unequal byte counts
                    (!dp.uniform_len && (uint64_t)dp.host.max_step_units * unit >= kDynSyncMinUneven)) &&
                   c->force_sync != 0) {
            // multi-step dynamic mode: queues per step, a CTA barrier per GPU row between steps,
            // one flag per peer GPU (the flow-ownership rule no longer applies)
            const TmaConfig tm = c->force_big > 0 ? kTmaBig : kTmaMid;
            E.stages = tm.stages;
            E.chunk = tm.chunk;
            E.ahead = tm.ahead;
            nC = c->force_big > 0 ? c->cap_big : c->cap_ctas;
            const uint64_t total = (uint64_t)dp.host.max_step_units * unit;
            uint64_t U = total / ((uint64_t)nC * (uint64_t)c->dyn_pieces);
            U = std::max<uint64_t>((uint64_t)E.chunk, std::min<uint64_t>(U, kDynMaxPiece));
            U = U / (uint64_t)E.chunk * (uint64_t)E.chunk;
            E.nS = nC;
            E.nF = 1;
            E.dyn_units = (int32_t)dp.dyn_tiles;
            E.dyn_u = (int32_t)U;
            E.dyn_sync = 1;
        }
        // several GPUs: CTAs of a GPU meet at a GPU-scope counter barrier after each step and ONE
        // system-scope release per peer GPU signals it, instead of one per (CTA, peer): 296 CTAs
        // x (G-1) peers of microsecond releases per step otherwise (measured, 8 emulated GPUs:
        // ring allgather 16 KiB 341 -> 285 us, Bruck allgather 64 KiB 125 -> 102 us; single-step
        // launches unchanged)
        if (c->G > 1 && c->row_signal) {
            // (and the CTAs split the GPU's own moves evenly: the kernel's flow-group ranges
            // become move-index ranges, so step 0's flow-range prefetch does not apply)
            if (!E.dyn_units) E.d0_base = -1;
            E.dyn_sync = 1;
        }
        // warp-ring dynamic mode: when some moves may not be 16-B congruent, every warp streams
        // its own pieces through a TMA ring -- congruent ones with bulk stores, the others with
        // 16-B stores the warp shifts out of shared memory (exec_kernel.cu dyn_tile_w; measured,
        // cfg4 mean 4 MiB int64: 96.9 / 103.1 / 106.6 -> 92.3 / 87.2 / 100.6 us, seeds 0-2)
        // (measured, cfg4 int64, first version: the LSU path won below ~100 MiB per GPU -- mean
        // 1 MiB 24.3 vs 25.7 us -- and the warp rings above: mean 2 MiB 55.5 -> 51.9, 4 MiB 96.9
        // -> 92.3; with constant-shift stores the rings win from 1 MiB: kWringMinVol)
        const uint64_t wr_vol = dp.nsteps == 1 ? src_vol : step_vol;
        if (E.dyn_units && c->wring &&
            (c->wring == 2 ||
             (wr_vol >= kWringMinVol &&
              (unit % 16 || ((uintptr_t)send | (uintptr_t)recv | send_stride | recv_stride | E.work_stride) % 16)))) {
            E.wring = 1;
            E.wslack = c->wslack;
            E.chunk = kWChunk;
            E.stages = kWarpsExec * kWStages;   // dynamic smem = stages x chunk (every warp's ring)
            E.ahead = 0;
            if (dp.nsteps == 1) {
                // queue pieces: the same share per CTA as above, but rounded to the nearest warp
                // chunk (4 KiB) instead of down to a 16 KiB ring chunk -- e.g. 28 instead of 16
                // KiB at cfg4 mean 8 MiB (measured: mean 6 / 8 MiB 124.7 / 165.6 -> 123.3 / 162.3
                // us, seed 1 162.3 -> 156.9; 2 / 4 MiB unchanged; 4 / 8 KiB pieces much slower)
                uint64_t U = src_vol / ((uint64_t)nC * (uint64_t)c->dyn_pieces);
                U = std::max<uint64_t>(kWringMinPiece, std::min<uint64_t>(U, kDynMaxPiece));
                // larger piece floors from 192 / 256 MiB per GPU: 20 / 24 KiB instead of the 16 /
                // 17 KiB shares of cfg4 means 4 / 5 MiB (the mean-4 MiB matrices total 250-256 MiB,
                // so they take the 20 KiB floor) -- measured, int64 seeds 0 / 1: 86.7 / 83.5 -> 85.4
                // / 82.0 us at 4 MiB, 100.7 / 100.6 -> 99.7 / 99.2 at 5 MiB; int32 the same; 3 / 6
                // MiB neutral, 8 MiB shares 28 KiB (profiles/r02/cfg4_pieces_s19.txt; the s21 build
                // with the 24 KiB floor alone left mean 4 MiB at 16 KiB pieces: 85.8 us in bench)
                if (src_vol >= kWringFloorVol24) U = std::max<uint64_t>(U, 24u << 10);
                else if (src_vol >= kWringFloorVol20) U = std::max<uint64_t>(U, 20u << 10);
                if (ntiles >= 4) U = std::max<uint64_t>(U, 3 * (uint64_t)kTmaMid.chunk);   // (as above)
                E.dyn_u = (int32_t)((U + kWChunk / 2) / kWChunk * kWChunk);
            }
        }
        // pre-wait L2 prefetch of the grid's first pieces (one GPU; kernel prologue): one piece
        // per CTA for the producer ring (allgather 4 / 64 MiB 56.1 / 746.4 -> 54.0 / 744.6 us,
        // alltoall 4 MiB blocks 83.0 -> 82.5), one per warp for the warp rings (cfg4 mean 2 / 4
        // MiB 48.6 / 88.2 -> 47.0 / 87.2 us; two per warp or one per CTA: no better)
        // (profiles/r02/prewait_l2_ab.txt)
        if (E.dyn_units && c->G == 1 && c->nprocs == 1 && c->prefetch)
            E.dyn_prefetch = E.wring ? kWarpsExec : 1;
        coop = coop_level(c, dp.nsteps > 1 && nC > 1);
        e = launch_exec(E, nC, c->emulated ? c->G : 1, coop, pdl && c->pdl, stream);
    }
    if (e != cudaSuccess) {
        if (getenv("MPXA_DEBUG")) fprintf(stderr, "mpxa: launch failed: %s\n", cudaGetErrorString(e));
        return MPXA_ERR_CUDA;
    }
    c->launches++;
    // execution path of this launch (tests assert the intended path ran: mpxa__last_launch)
    c->last_path = (small ? 1u : 0u) | (E.small_ll ? 2u : 0u) | (E.small_var ? 4u : 0u) |
                   (E.dyn_units ? 8u : 0u) | (E.dyn_sync ? 16u : 0u) | (E.small_own ? 32u : 0u) |
                   (E.small_swork ? 64u : 0u) | (E.wring ? 128u : 0u) | (tiny ? 256u : 0u) |
                   (coop ? 512u : 0u);
    return MPXA_SUCCESS;
}

// per-call program upload through a ring of pinned slots (stream-ordered, no host sync
// unless the ring wraps onto a copy still in flight)
int run_dynamic(mpxa_comm_t c, const Program &P, const char *send, char *recv, uint64_t unit,
                uint64_t send_stride, uint64_t recv_stride, cudaStream_t stream) {
    if (c->ring.empty()) c->ring.resize(8);
    Slot &s = c->ring[c->ring_next];
    c->ring_next = (c->ring_next + 1) % (int)c->ring.size();
    if (!s.ev) CK(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
    if (s.used) CK(cudaEventSynchronize(s.ev));
    size_t n = serialized_size(P);
    if (n > s.cap) {
        if (s.dmem) CK(cudaFree(s.dmem));
        CK(cudaMalloc(&s.dmem, n));
        s.cap = n;
    }
    if (n > s.pcap) {
        if (s.pinned) CK(cudaFreeHost(s.pinned));
        CK(cudaHostAlloc((void **)&s.pinned, n, cudaHostAllocDefault));
        s.pcap = n;
    }
    std::vector<char> buf;
    serialize(P, buf, (uintptr_t)s.dmem);
    memcpy(s.pinned, buf.data(), n);
    CK(cudaMemcpyAsync(s.dmem, s.pinned, n, cudaMemcpyHostToDevice, stream));
    DevProg dp;
    dp.per_call = true;
    dp.dmem = s.dmem;
    dp.gp.assign((const GpuProg *)buf.data(), (const GpuProg *)buf.data() + P.G);
    dp.bytes = n;
    dp.host = P;
    dp.nsteps = P.nsteps();
    prog_facts(dp);
    int rc = run_program(c, dp, send, recv, unit, send_stride, recv_stride, stream, nullptr, /*pdl=*/false);
    CK(cudaEventRecord(s.ev, stream));
    s.used = true;
    dp.dmem = nullptr;
    return rc;
}

}  // namespace mpxa_rt

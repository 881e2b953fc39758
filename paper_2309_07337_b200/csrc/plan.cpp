// Schedule builders.  Each builder emits the steps of
// the paper-family algorithm as moves executed by the GPU that owns the SOURCE rank (push
// model: payload crosses NVLink as stores into the peer's buffer).  A move never
// concatenates units that later moves split, so the column slice a CTA owns is the same
// byte range of a block in every step (mpxa_exec_kernel's ownership rule).
#include "plan.h"

#include <algorithm>
#include <cstdlib>
#include <map>

#include "../../include/mpxa.h"

namespace mpxa {

int ceil_log2(int p) {
    int k = 0;
    while ((1 << k) < p) k++;
    return k;
}

static inline int imod(int64_t a, int p) {
    int64_t r = a % p;
    return (int)(r < 0 ? r + p : r);
}

namespace {

class Builder {
public:
    Builder(Program &P, int p, int R, int G, int nflows) : P_(P), p_(p), R_(R), G_(G) {
        P_ = Program();
        P_.p = p; P_.R = R; P_.G = G;
        P_.nflows = nflows;
        P_.steps.assign(G, {});
        P_.moves.assign(G, {});
        P_.findex.assign(G, {});
        cur_.assign(G, {});
    }
    // flow < 0: the flow of the data currently at the source location (set by the move
    // that wrote it); SEND-sourced moves pass their origin flow explicitly.
    void move(int sk, int sr, int64_t so, int dk, int dr, int64_t dof, int64_t len, int64_t flow = -1,
              int fan = 0) {
        if (len <= 0) return;
        if (flow < 0) {
            auto it = loc_.find(key(sk, sr, so));
            flow = it == loc_.end() ? 0 : it->second;
        }
        Move m{};
        m.src_off = so; m.dst_off = dof; m.len = len;
        m.flow = (uint32_t)flow;
        m.src_rank = (uint16_t)sr; m.dst_rank = (uint16_t)dr;
        m.src_kind = (uint8_t)sk; m.dst_kind = (uint8_t)dk; m.fanout = (uint8_t)fan;
        cur_[sr / R_].push_back(m);
        if (!fan) pending_.push_back({key(dk, dr, dof), (uint32_t)flow});
    }
    void end_step() {
        for (auto &kv : pending_) loc_[kv.first] = kv.second;
        pending_.clear();
        bool any = false;                       // a step without moves on every GPU is dropped
        for (int g = 0; g < G_ && !any; g++) any = !cur_[g].empty();
        if (!any) return;
        std::vector<uint32_t> sig(G_, 0), wt(G_, 0);
        for (int g = 0; g < G_; g++)
            for (const Move &m : cur_[g]) {
                if (m.fanout) {
                    for (int d = 0; d < G_; d++)
                        if (d != g) { sig[g] |= 1u << d; wt[d] |= 1u << g; }
                } else {
                    int d = m.dst_rank / R_;
                    if (d != g) { sig[g] |= 1u << d; wt[d] |= 1u << g; }
                }
            }
        for (int g = 0; g < G_; g++) {
            std::stable_sort(cur_[g].begin(), cur_[g].end(),
                             [](const Move &a, const Move &b) { return a.flow < b.flow; });
            Step s{};
            s.move_begin = (int32_t)P_.moves[g].size();
            int64_t tot = 0, mx = 0;
            for (const Move &m : cur_[g]) {
                P_.moves[g].push_back(m);
                tot += m.len * (m.fanout ? p_ : 1);
                mx = std::max(mx, m.len);
            }
            s.move_end = (int32_t)P_.moves[g].size();
            s.signal_mask = sig[g];
            s.wait_mask = wt[g];
            s.total_len = tot;
            s.max_len = mx;
            s.flow_index = (int32_t)P_.findex[g].size();
            s.dense_base = -1;
            if (!cur_[g].empty()) {
                bool dense = true;
                const uint32_t fb = cur_[g][0].flow;
                for (size_t k = 0; k < cur_[g].size() && dense; k++) dense = cur_[g][k].flow == fb + (uint32_t)k;
                if (dense) s.dense_base = (int32_t)fb;
            }
            size_t q = 0;
            for (int x = 0; x <= P_.nflows; x++) {       // findex[x] = #moves with flow < x
                while (q < cur_[g].size() && cur_[g][q].flow < (uint32_t)x) q++;
                P_.findex[g].push_back((int32_t)q);
            }
            P_.steps[g].push_back(s);
            P_.max_move = std::max(P_.max_move, mx);
            P_.max_step_units = std::max(P_.max_step_units, tot);
            P_.max_step_moves = std::max<int64_t>(P_.max_step_moves, (int64_t)cur_[g].size());
            P_.signals += __builtin_popcount(sig[g]);
            cur_[g].clear();
        }
    }

private:
    static uint64_t key(int k, int r, int64_t off) {
        return ((uint64_t)k << 62) ^ ((uint64_t)r << 44) ^ (uint64_t)off;
    }
    Program &P_;
    int p_, R_, G_;
    std::vector<std::vector<Move>> cur_;
    std::unordered_map<uint64_t, uint32_t> loc_;
    std::vector<std::pair<uint64_t, uint32_t>> pending_;
};

bool topo_ok(int p, int R, int G) {
    return p >= 1 && R >= 1 && G >= 1 && G <= kMaxGpus && p == R * G && p <= 65535;
}

}  // namespace

// ---------------------------------------------------------------------------------------
// alltoall
// ---------------------------------------------------------------------------------------
bool build_alltoall(Program &P, int algo, int p, int R, int G, int g, int stop_stage, bool hier_staged) {
    if (!topo_ok(p, R, G)) return false;
    Builder B(P, p, R, G, p * p);
    if (algo == A_PAIRWISE) {
        // A3: step s sends to (r+s) mod p; all s run concurrently on the GPU.
        for (int s = 0; s < p; s++)
            for (int t = 0; t < p; t++) {
                int j = imod(s + t, p);
                B.move(BK_SEND, s, j, BK_RECV, j, s, 1, (int64_t)s * p + j);
            }
        B.end_step();
        P.work_units = 0;
        return true;
    }
    if (algo == A_BRUCK) {
        // A4-A6: T_r[i] = send_r[(r+i) mod p]; round k: the blocks with bit k of i set go, in
        // increasing i, to (r+2^k) mod p, which keeps them as its new T[i]; finally
        // recv_r[j] = T_r[(r-j) mod p].  The rotation is virtual: a block that has not moved
        // yet is READ from send_r[(r+i) mod p] where round k (or the inverse rotation) needs
        // it -- no HBM pass for A4.  Zero-copy receive: round k lands in the receiver's round-k
        // area S_k and T[i] is thereafter read from there (loc[i]) instead of being unpacked
        // over the old T[i].  Every workspace byte is written once per launch, so no CTA ever
        // overwrites data another CTA has still to read.
        const int K = ceil_log2(p);
        std::vector<int64_t> soff(K + 1, 0);
        for (int k = 0; k < K; k++) {
            int64_t mk = 0;
            for (int i = 0; i < p; i++) mk += (i >> k) & 1;
            soff[k + 1] = soff[k] + mk;
        }
        P.work_units = soff[K];
        std::vector<int64_t> loc(p, -1);                     // WORK offset of T[i]; -1: still in send
        // T_r[i] read where it currently is (rank r's send buffer, rotated, or its WORK row)
        auto read_T = [&](int r, int i, int dk, int dr, int64_t dof) {
            if (loc[i] < 0) {
                const int b = imod(r + i, p);
                B.move(BK_SEND, r, b, dk, dr, dof, 1, (int64_t)r * p + b);
            } else {
                B.move(BK_WORK, r, loc[i], dk, dr, dof, 1);
            }
        };
        const int rounds = stop_stage < 0 ? K : std::min(stop_stage, K);
        for (int k = 0; k < rounds; k++) {                   // A5 bit-indexed rounds
            const int d = 1 << k;
            for (int r = 0; r < p; r++) {
                int64_t pos = 0;
                for (int i = 0; i < p; i++)
                    if ((i >> k) & 1) read_T(r, i, BK_WORK, imod(r + d, p), soff[k] + pos++);
            }
            B.end_step();
            int64_t pos = 0;
            for (int i = 0; i < p; i++)
                if ((i >> k) & 1) loc[i] = soff[k] + pos++;
        }
        if (stop_stage < 0) {                                // A6 inverse rotation
            for (int r = 0; r < p; r++)
                for (int j = 0; j < p; j++) read_T(r, imod(r - j, p), BK_RECV, r, j);
        } else {                                             // dump T for stage tests
            for (int r = 0; r < p; r++)
                for (int i = 0; i < p; i++) read_T(r, i, BK_RECV, r, i);
        }
        B.end_step();
        return true;
    }
    if (algo == A_HIER) {
        if (g < 1 || p % g) return false;
        std::vector<int64_t> c((size_t)p * p, 1), sd((size_t)p * p), rd((size_t)p * p);
        for (int s = 0; s < p; s++)
            for (int j = 0; j < p; j++) { sd[(size_t)s * p + j] = j; rd[(size_t)j * p + s] = s; }
        return build_alltoallv(P, A_HIER, p, R, G, g, c.data(), sd.data(), rd.data(), hier_staged);
    }
    return false;
}

// ---------------------------------------------------------------------------------------
// allgather
// ---------------------------------------------------------------------------------------
bool build_allgather(Program &P, int algo, int p, int R, int G, int stop_stage, int gsize) {
    if (!topo_ok(p, R, G)) return false;
    Builder B(P, p, R, G, p);
    if (algo == A_PAIRWISE) {
        // direct: read send_s once, store it into block s of every rank's recvbuf
        for (int s = 0; s < p; s++) B.move(BK_SEND, s, 0, BK_RECV, 0, s, 1, s, /*fanout=*/1);
        B.end_step();
        return true;
    }
    if (algo == A_RING) {
        // recv_r[r] = send_r; step s: r sends block (r-s) mod p to r+1.
        for (int r = 0; r < p; r++) {
            B.move(BK_SEND, r, 0, BK_RECV, r, r, 1, r);
            if (p > 1) B.move(BK_SEND, r, 0, BK_RECV, imod(r + 1, p), r, 1, r);
        }
        B.end_step();
        for (int s = 1; s < p - 1; s++) {
            for (int r = 0; r < p; r++) {
                int b = imod(r - s, p);
                B.move(BK_RECV, r, b, BK_RECV, imod(r + 1, p), b, 1);
            }
            B.end_step();
        }
        return true;
    }
    if (algo == A_HIER) {
        // f2(i) locality-aware allgather over groups of g ranks (default: the ranks of one
        // GPU): every block crosses each group boundary ONCE -- step 1 sends it to the ranks of
        // its own group and to one receiver in each remote group B, rank B*g + (A mod g)
        // (SPEC.md:161's leader rotation), straight into that rank's recvbuf; step 2 that
        // receiver replicates it to the other ranks of B.  (SPEC.md:233 gathers to one leader
        // and runs Bruck among leaders; on NVSwitch every group is one hop away, so the inter-
        // group step is a direct exchange -- same result.)
        const int g = gsize;
        if (g < 1 || p % g) return false;
        const int NG = p / g;
        for (int r = 0; r < p; r++) {
            const int A = r / g;
            for (int t = 0; t < g; t++) B.move(BK_SEND, r, 0, BK_RECV, A * g + t, r, 1, r);
            for (int Bg = 0; Bg < NG; Bg++)
                if (Bg != A) B.move(BK_SEND, r, 0, BK_RECV, Bg * g + (A % g), r, 1, r);
        }
        B.end_step();
        for (int r = 0; r < p; r++) {
            const int A = r / g;
            for (int Bg = 0; Bg < NG; Bg++) {
                if (Bg == A) continue;
                const int lead = Bg * g + (A % g);
                for (int t = 0; t < g; t++)
                    if (Bg * g + t != lead) B.move(BK_RECV, lead, r, BK_RECV, Bg * g + t, r, 1);
            }
        }
        B.end_step();
        return true;
    }
    if (algo == A_BRUCK) {
        // T_r[0] = send_r; round k sends T_r[0..n_k) to (r-2^k) mod p,
        // stored at T[2^k..2^k+n_k); recv_r[j] = T_r[(j-r) mod p].  T_r[0] is never copied:
        // it is read from send_r wherever it is needed (WORK row 0 stays unused).
        const int K = ceil_log2(p);
        P.work_units = p;
        auto read_T = [&](int r, int i, int dk, int dr, int64_t dof) {
            if (i == 0) B.move(BK_SEND, r, 0, dk, dr, dof, 1, r);
            else B.move(BK_WORK, r, i, dk, dr, dof, 1);
        };
        const int rounds = stop_stage < 0 ? K : std::min(stop_stage, K);
        for (int k = 0; k < rounds; k++) {
            const int d = 1 << k, nk = std::min(d, p - d);
            for (int r = 0; r < p; r++)
                for (int i = 0; i < nk; i++) read_T(r, i, BK_WORK, imod(r - d, p), d + i);
            B.end_step();
        }
        if (stop_stage < 0) {
            for (int r = 0; r < p; r++)
                for (int j = 0; j < p; j++) read_T(r, imod(j - r, p), BK_RECV, r, j);
        } else {
            int filled = std::min(1 << rounds, p);
            for (int r = 0; r < p; r++)
                for (int i = 0; i < filled; i++) read_T(r, i, BK_RECV, r, i);
        }
        B.end_step();
        return true;
    }
    return false;
}

// ---------------------------------------------------------------------------------------
// alltoallv
// ---------------------------------------------------------------------------------------
bool build_alltoallv(Program &P, int algo, int p, int R, int G, int g, const int64_t *c,
                     const int64_t *sd, const int64_t *rd, bool hier_staged) {
    if (!topo_ok(p, R, G)) return false;
    auto C = [&](int s, int j) { return c[(size_t)s * p + j]; };
    auto SD = [&](int s, int j) { return sd[(size_t)s * p + j]; };
    auto RD = [&](int j, int s) { return rd[(size_t)j * p + s]; };
    if (algo == A_PAIRWISE) {
        Builder B(P, p, R, G, p * p);
        for (int s = 0; s < p; s++)
            for (int t = 0; t < p; t++) {
                int j = imod(s + t, p);
                B.move(BK_SEND, s, SD(s, j), BK_RECV, j, RD(j, s), C(s, j), (int64_t)s * p + j);
            }
        B.end_step();
        P.work_units = 0;
        return true;
    }
    if (algo == A_BRUCK) {
        // f2(iii) Bruck alltoallv (north_star "Bruck ... pack/unpack for ... v-variants"; paper
        // silent): A4-A6 with per-rank variable blocks.  T_r[i] starts as the
        // segment r sends to (r+i) mod p; round k moves the blocks with bit k of i to (r+2^k)
        // mod p, landing in that rank's round-k area (zero-copy receive, as for alltoall);
        // finally recv_r[rd_r[j]] = T_r[(r-j) mod p].  Areas are sized per rank.
        Builder B(P, p, R, G, p * p);
        const int K = ceil_log2(p);
        // loc[r][i] < 0: T_r[i] has not moved and is read from rank r's send buffer (the
        // rotation is virtual, as for alltoall); else its offset in rank r's WORK row
        std::vector<std::vector<int64_t>> loc(p, std::vector<int64_t>(p, -1)), len(p, std::vector<int64_t>(p));
        std::vector<int64_t> cur(p, 0);
        for (int r = 0; r < p; r++)
            for (int i = 0; i < p; i++) len[r][i] = C(r, imod(r + i, p));
        auto read_T = [&](int r, int i, int dk, int dr, int64_t dof) {
            if (loc[r][i] < 0) {
                const int j = imod(r + i, p);
                B.move(BK_SEND, r, SD(r, j), dk, dr, dof, len[r][i], (int64_t)r * p + j);
            } else {
                B.move(BK_WORK, r, loc[r][i], dk, dr, dof, len[r][i]);
            }
        };
        for (int k = 0; k < K; k++) {                        // A5 rounds
            const int d = 1 << k;
            std::vector<std::vector<int64_t>> nloc = loc, nlen = len;
            for (int r = 0; r < p; r++) {
                const int to = imod(r + d, p);
                for (int i = 0; i < p; i++)
                    if ((i >> k) & 1) {
                        read_T(r, i, BK_WORK, to, cur[to]);
                        nloc[to][i] = cur[to];
                        nlen[to][i] = len[r][i];
                        cur[to] += len[r][i];
                    }
            }
            B.end_step();
            loc.swap(nloc);
            len.swap(nlen);
        }
        for (int r = 0; r < p; r++)                          // A6 inverse rotation
            for (int j = 0; j < p; j++) {
                const int i = imod(r - j, p);
                if (len[r][i] != C(j, r)) return false;      // (counts consistent by construction)
                read_T(r, i, BK_RECV, r, RD(r, j));
            }
        B.end_step();
        int64_t work = 0;
        for (int r = 0; r < p; r++) work = std::max(work, cur[r]);
        P.work_units = work;
        return true;
    }
    if (algo != A_HIER) return false;
    if (g < 1 || p % g) return false;
    if (g == R && !hier_staged) {
        // A8 with group = GPU, fused ("steps 1 and 3 are HBM-local and can be
        // fused into K1's addressing"): the GPU of group A reads every local rank's segments
        // for group B and stores them straight into B's ranks' recvbufs -- one aggregated
        // transfer per GPU pair carrying one flag per CTA, i.e. the G(G-1) inter-group
        // messages of the staged form without its two HBM-local passes.
        Builder B(P, p, R, G, p * p);
        for (int s = 0; s < p; s++)
            for (int t = 0; t < p; t++) {
                int j = imod(s + t, p);
                B.move(BK_SEND, s, SD(s, j), BK_RECV, j, RD(j, s), C(s, j), (int64_t)s * p + j);
            }
        B.end_step();
        P.work_units = 0;
        return true;
    }
    // A8: groups of g consecutive ranks, leader
    // L(A,B) = A*g + (B mod g); aggregated message segments ordered (s,t) row-major.
    const int NG = p / g;
    auto L = [&](int A, int Bg) { return A * g + (Bg % g); };
    auto pair_units = [&](int A, int Bg) {
        int64_t n = 0;
        for (int s = 0; s < g; s++)
            for (int t = 0; t < g; t++) n += C(A * g + s, Bg * g + t);
        return n;
    };
    // work layout of every rank: first the out-aggregates it leads, then the in-aggregates
    std::vector<int64_t> out_off((size_t)NG * NG, -1), in_off((size_t)NG * NG, -1);
    int64_t work = 0;
    for (int x = 0; x < p; x++) {
        int64_t cur = 0;
        int A = x / g;
        for (int Bg = 0; Bg < NG; Bg++)
            if (Bg != A && L(A, Bg) == x) { out_off[(size_t)A * NG + Bg] = cur; cur += pair_units(A, Bg); }
        for (int A2 = 0; A2 < NG; A2++)   // x receives pair (A2 -> A) when L(A, A2) == x
            if (A2 != A && L(A, A2) == x) { in_off[(size_t)A2 * NG + A] = cur; cur += pair_units(A2, A); }
        work = std::max(work, cur);
    }
    auto segoff = [&](int A, int Bg, int s, int t) {
        int64_t o = 0;
        for (int s2 = 0; s2 < g; s2++)
            for (int t2 = 0; t2 < g; t2++) {
                if (s2 == s && t2 == t) return o;
                o += C(A * g + s2, Bg * g + t2);
            }
        return o;
    };
    Builder B(P, p, R, G, p * p);
    P.work_units = work;
    // step 1: intra-group direct + gather to leaders
    for (int r = 0; r < p; r++) {
        int A = r / g, s = r % g;
        for (int t = 0; t < g; t++) {
            int j = A * g + t;
            B.move(BK_SEND, r, SD(r, j), BK_RECV, j, RD(j, r), C(r, j), (int64_t)r * p + j);
        }
        for (int Bg = 0; Bg < NG; Bg++) {
            if (Bg == A) continue;
            int lead = L(A, Bg);
            for (int t = 0; t < g; t++) {
                int j = Bg * g + t;
                B.move(BK_SEND, r, SD(r, j), BK_WORK, lead, out_off[(size_t)A * NG + Bg] + segoff(A, Bg, s, t), C(r, j),
                       (int64_t)r * p + j);
            }
        }
    }
    B.end_step();
    // step 2: one aggregated exchange per group pair (segment-wise moves, one signal)
    for (int A = 0; A < NG; A++)
        for (int Bg = 0; Bg < NG; Bg++) {
            if (Bg == A) continue;
            int lead = L(A, Bg), peer = L(Bg, A);
            for (int s = 0; s < g; s++)
                for (int t = 0; t < g; t++) {
                    int64_t o = segoff(A, Bg, s, t);
                    B.move(BK_WORK, lead, out_off[(size_t)A * NG + Bg] + o, BK_WORK, peer,
                           in_off[(size_t)A * NG + Bg] + o, C(A * g + s, Bg * g + t));
                }
        }
    B.end_step();
    // step 3: redistribute segment (s,t) to rank Bg*g+t at rdispls[A*g+s]
    for (int Bg = 0; Bg < NG; Bg++)
        for (int A = 0; A < NG; A++) {
            if (A == Bg) continue;
            int lead = L(Bg, A);
            for (int s = 0; s < g; s++)
                for (int t = 0; t < g; t++) {
                    int dst = Bg * g + t, src = A * g + s;
                    B.move(BK_WORK, lead, in_off[(size_t)A * NG + Bg] + segoff(A, Bg, s, t), BK_RECV, dst,
                           RD(dst, src), C(src, dst));
                }
        }
    B.end_step();
    return true;
}

// ---------------------------------------------------------------------------------------
// f1: persistent neighborhood alltoallv (§2.2)
// ---------------------------------------------------------------------------------------
namespace {

struct NbGraph {
    int p;
    std::vector<int64_t> ioff, ooff, ie, oe;   // edge offsets per rank; element offsets per edge
    std::vector<int64_t> match;                // in-edge -> matched global out-edge
};

// Validates the graph (valid ranks, non-negative counts / displacements, MPI pairing with equal
// counts, every out-edge paired) and pairs the edges.
int nb_prepare(NbGraph &N, int p, const int *indeg, const int *src, const int64_t *rc, const int64_t *rd,
               const int *outdeg, const int *dst, const int64_t *sc, const int64_t *sd) {
    N.p = p;
    N.ioff.assign(p + 1, 0);
    N.ooff.assign(p + 1, 0);
    for (int r = 0; r < p; r++) {
        if (indeg[r] < 0 || outdeg[r] < 0) return MPXA_ERR_ARG;
        N.ioff[r + 1] = N.ioff[r] + indeg[r];
        N.ooff[r + 1] = N.ooff[r] + outdeg[r];
    }
    const int64_t ni = N.ioff[p], no = N.ooff[p];
    if (ni != no) return MPXA_ERR_MISMATCH;
    for (int64_t e = 0; e < ni; e++)
        if (src[e] < 0 || src[e] >= p || rc[e] < 0 || rd[e] < 0) return MPXA_ERR_ARG;
    for (int64_t e = 0; e < no; e++)
        if (dst[e] < 0 || dst[e] >= p || sc[e] < 0 || sd[e] < 0) return MPXA_ERR_ARG;
    N.ie.assign(ni + 1, 0);
    N.oe.assign(no + 1, 0);
    for (int64_t e = 0; e < ni; e++) N.ie[e + 1] = N.ie[e] + rc[e];
    for (int64_t e = 0; e < no; e++) N.oe[e + 1] = N.oe[e] + sc[e];
    // pair: per (r, q), the k-th out-edge r->q with the k-th in-edge q<-r
    std::map<std::pair<int, int>, std::vector<int64_t>> outs;
    for (int r = 0; r < p; r++)
        for (int64_t e = N.ooff[r]; e < N.ooff[r + 1]; e++) outs[{r, dst[e]}].push_back(e);
    std::map<std::pair<int, int>, size_t> used;
    N.match.assign(ni, -1);
    for (int q = 0; q < p; q++)
        for (int64_t e = N.ioff[q]; e < N.ioff[q + 1]; e++) {
            auto key = std::make_pair(src[e], q);
            size_t k = used[key]++;
            auto it = outs.find(key);
            if (it == outs.end() || k >= it->second.size()) return MPXA_ERR_MISMATCH;
            const int64_t o = it->second[k];
            if (sc[o] != rc[e]) return MPXA_ERR_MISMATCH;
            N.match[e] = o;
        }
    for (auto &kv : outs)
        if (used[kv.first] != kv.second.size()) return MPXA_ERR_MISMATCH;
    return MPXA_SUCCESS;
}

}  // namespace

int build_neighbor(Program &P, bool locality, int p, int R, int G, int g, const int *indeg, const int *src,
                   const int64_t *rc, const int64_t *rd, const int *outdeg, const int *dst, const int64_t *sc,
                   const int64_t *sd, const int64_t *send_idx, const int64_t *recv_idx, bool staged) {
    if (!topo_ok(p, R, G)) return MPXA_ERR_TOPOLOGY;
    NbGraph N;
    int rcode = nb_prepare(N, p, indeg, src, rc, rd, outdeg, dst, sc, sd);
    if (rcode) return rcode;
    const int64_t no = N.ooff[p];
    if (!locality) {
        // standard: one move per out-edge with a count, sender side
        Builder B(P, p, R, G, (int)std::max<int64_t>(1, no));
        for (int q = 0; q < p; q++)
            for (int64_t e = N.ioff[q]; e < N.ioff[q + 1]; e++) {
                const int64_t o = N.match[e];
                B.move(BK_SEND, src[e], sd[o], BK_RECV, q, rd[e], rc[e], o);
            }
        B.end_step();
        P.work_units = 0;
        return MPXA_SUCCESS;
    }
    // locality-aware three-phase plan over groups of g ranks
    if (g < 1 || p % g) return MPXA_ERR_TOPOLOGY;
    if ((N.oe[no] && !send_idx) || (N.ie[N.ioff[p]] && !recv_idx)) return MPXA_ERR_ARG;
    for (int q = 0; q < p; q++)              // index handshake: received ids = matched sent ids
        for (int64_t e = N.ioff[q]; e < N.ioff[q + 1]; e++) {
            const int64_t o = N.match[e];
            for (int64_t x = 0; x < rc[e]; x++)
                if (recv_idx[N.ie[e] + x] != send_idx[N.oe[o] + x]) return MPXA_ERR_TOPOLOGY;
        }
    auto L = [&](int A, int Bg) { return A * g + (Bg % g); };
    const int NG = p / g;
    // per group pair (A,B): unique ids (sorted), the first holder (rank, element offset in its
    // sendbuf) of each in (rank, edge, element) order, and every final destination (rank,
    // element offset in its recvbuf) in receiver element order
    struct SrcEl { int64_t id, off; int r; };
    struct DstEl { int64_t slot, off; int q; };
    struct PairSched {
        std::vector<int64_t> ids, hoff;
        std::vector<int> holder;
        std::vector<DstEl> dests;          // sorted by slot (stable: receiver order inside)
        std::vector<int64_t> dstart;       // dests of slot s: [dstart[s], dstart[s+1])
    };
    std::vector<PairSched> ps((size_t)NG * NG);
    {
        std::vector<std::vector<SrcEl>> sends((size_t)NG * NG);
        for (int r = 0; r < p; r++)
            for (int64_t o = N.ooff[r]; o < N.ooff[r + 1]; o++) {
                const int A = r / g, Bg = dst[o] / g;
                if (A == Bg) continue;
                auto &v = sends[(size_t)A * NG + Bg];
                for (int64_t x = 0; x < sc[o]; x++) v.push_back(SrcEl{send_idx[N.oe[o] + x], sd[o] + x, r});
            }
        for (size_t k = 0; k < sends.size(); k++) {
            auto &v = sends[k];
            std::stable_sort(v.begin(), v.end(), [](const SrcEl &x, const SrcEl &y) { return x.id < y.id; });
            PairSched &P2 = ps[k];
            for (size_t i = 0; i < v.size(); i++)
                if (i == 0 || v[i].id != v[i - 1].id) {   // first holder of each id
                    P2.ids.push_back(v[i].id);
                    P2.hoff.push_back(v[i].off);
                    P2.holder.push_back(v[i].r);
                }
        }
    }
    for (int q = 0; q < p; q++)
        for (int64_t e = N.ioff[q]; e < N.ioff[q + 1]; e++) {
            const int A = src[e] / g, Bg = q / g;
            if (A == Bg) continue;
            PairSched &P2 = ps[(size_t)A * NG + Bg];
            for (int64_t x = 0; x < rc[e]; x++) {
                const int64_t id = recv_idx[N.ie[e] + x];
                const int64_t slot = std::lower_bound(P2.ids.begin(), P2.ids.end(), id) - P2.ids.begin();
                P2.dests.push_back(DstEl{slot, rd[e] + x, q});
            }
        }
    for (PairSched &P2 : ps) {
        std::stable_sort(P2.dests.begin(), P2.dests.end(), [](const DstEl &x, const DstEl &y) { return x.slot < y.slot; });
        P2.dstart.assign(P2.ids.size() + 1, 0);
        for (const DstEl &d : P2.dests) P2.dstart[(size_t)d.slot + 1]++;
        for (size_t s2 = 0; s2 < P2.ids.size(); s2++) P2.dstart[s2 + 1] += P2.dstart[s2];
    }
    // runs: consecutive slots moved as one unit through all three steps -- same holder with
    // consecutive offsets and the same destination pattern shifted by one element
    struct Run { int A, Bg; size_t s0, n; };
    std::vector<Run> runs;
    for (int A = 0; A < NG; A++)
        for (int Bg = 0; Bg < NG; Bg++) {
            const PairSched &P2 = ps[(size_t)A * NG + Bg];
            const size_t n = P2.ids.size();
            size_t s0 = 0;
            for (size_t s2 = 1; s2 <= n; s2++) {
                bool cont = s2 < n && P2.holder[s2] == P2.holder[s2 - 1] && P2.hoff[s2] == P2.hoff[s2 - 1] + 1 &&
                            P2.dstart[s2 + 1] - P2.dstart[s2] == P2.dstart[s2] - P2.dstart[s2 - 1];
                for (int64_t d = 0; cont && d < P2.dstart[s2 + 1] - P2.dstart[s2]; d++) {
                    const DstEl &x = P2.dests[(size_t)(P2.dstart[s2] + d)], &y = P2.dests[(size_t)(P2.dstart[s2 - 1] + d)];
                    cont = x.q == y.q && x.off == y.off + 1;
                }
                if (!cont) { runs.push_back(Run{A, Bg, s0, s2 - s0}); s0 = s2; }
            }
        }
    // fused (group = GPU, g == R): the gather to the leader is GPU-local, so the exchange reads
    // each run straight from its holder's sendbuf (same GPU as the leader) -- two steps, no
    // out-aggregates (as for the hierarchical alltoall)
    const bool fused = g == R && !staged;
    // workspace of each rank: out-aggregates it leads, then in-aggregates it receives
    std::vector<int64_t> out_base((size_t)NG * NG, 0), in_base((size_t)NG * NG, 0), cur(p, 0);
    for (int A = 0; A < NG && !fused; A++)
        for (int Bg = 0; Bg < NG; Bg++) {
            const size_t k = (size_t)A * NG + Bg;
            if (ps[k].ids.empty()) continue;
            out_base[k] = cur[L(A, Bg)];
            cur[L(A, Bg)] += (int64_t)ps[k].ids.size();
        }
    for (int A = 0; A < NG; A++)
        for (int Bg = 0; Bg < NG; Bg++) {
            const size_t k = (size_t)A * NG + Bg;
            if (ps[k].ids.empty()) continue;
            in_base[k] = cur[L(Bg, A)];
            cur[L(Bg, A)] += (int64_t)ps[k].ids.size();
        }
    int64_t work = 0;
    for (int x = 0; x < p; x++) work = std::max(work, cur[x]);
    // flows: intra-group edges first, then runs
    int64_t nintra = 0;
    for (int r = 0; r < p; r++)
        for (int64_t o = N.ooff[r]; o < N.ooff[r + 1]; o++) nintra += (r / g == dst[o] / g);
    Builder B(P, p, R, G, (int)std::max<int64_t>(1, nintra + (int64_t)runs.size()));
    P.work_units = work;
    // step 1: intra-group edges directly; one representative of each run to L(A,B)
    int64_t f = 0;
    for (int q = 0; q < p; q++)
        for (int64_t e = N.ioff[q]; e < N.ioff[q + 1]; e++)
            if (src[e] / g == q / g) B.move(BK_SEND, src[e], sd[N.match[e]], BK_RECV, q, rd[e], rc[e], f++);
    for (size_t k = 0; k < runs.size(); k++) {
        const Run &u = runs[k];
        const size_t pk = (size_t)u.A * NG + u.Bg;
        if (fused)   // holder's sendbuf -> L(B,A), each unique id once
            B.move(BK_SEND, ps[pk].holder[u.s0], ps[pk].hoff[u.s0], BK_WORK, L(u.Bg, u.A), in_base[pk] + (int64_t)u.s0,
                   (int64_t)u.n, nintra + (int64_t)k);
        else
            B.move(BK_SEND, ps[pk].holder[u.s0], ps[pk].hoff[u.s0], BK_WORK, L(u.A, u.Bg), out_base[pk] + (int64_t)u.s0,
                   (int64_t)u.n, nintra + (int64_t)k);
    }
    B.end_step();
    // step 2: L(A,B) -> L(B,A), each unique id once (one signal per GPU pair per CTA)
    for (const Run &u : runs) {
        if (fused) break;
        const size_t pk = (size_t)u.A * NG + u.Bg;
        B.move(BK_WORK, L(u.A, u.Bg), out_base[pk] + (int64_t)u.s0, BK_WORK, L(u.Bg, u.A), in_base[pk] + (int64_t)u.s0,
               (int64_t)u.n);
    }
    B.end_step();   // (an empty step is dropped)
    // step 3: fan out to every final (rank, offset)
    for (const Run &u : runs) {
        const size_t pk = (size_t)u.A * NG + u.Bg;
        const PairSched &P2 = ps[pk];
        for (int64_t d = P2.dstart[u.s0]; d < P2.dstart[u.s0 + 1]; d++)
            B.move(BK_WORK, L(u.Bg, u.A), in_base[pk] + (int64_t)u.s0, BK_RECV, P2.dests[(size_t)d].q,
                   P2.dests[(size_t)d].off, (int64_t)u.n);
    }
    B.end_step();
    (void)f;
    return MPXA_SUCCESS;
}

}  // namespace mpxa

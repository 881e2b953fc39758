// libmpxa host runtime: variant registry and the measured selector (§2.1;
// SPEC.md:239-247).
#include "runtime.h"

namespace mpxa_rt {

// ---- selector -------------------------------------------------------------------------
int default_algo(mpxa_comm_t c, int op, size_t bytes) {
    if (c->user_algo[op]) return c->user_algo[op];
    // the measured table first (bench.py --write-selector); the rules below are fallbacks for
    // configurations no table row covers -- they were NOT measured on NVLink
    for (const SelEntry &e : c->selector)
        if (e.op == op && e.p == c->p && e.R == c->R && (e.G < 0 || e.G == c->G) && (e.g < 0 || e.g == c->g) &&
            bytes <= e.max_bytes)
            return e.algo;
    // SPEC.md:256 defaults when nothing was measured: pairwise (alltoall/v: its flags are
    // already one per GPU pair and CTA, so the hierarchical variant's fewer messages buy
    // nothing here).  Allgather: the direct (pairwise) exchange -- except across GPUs with
    // several ranks per GPU beyond the eager range, where direct fan-out sends every block to
    // each of a peer GPU's R ranks over NVLink and the hierarchical variant (groups = GPUs,
    // SURVEY §8 A10 "hier when R > 1") sends it once per GPU: R x fewer NVLink bytes.
    if (op == MPXA_OP_ALLGATHER && c->G > 1 && c->Rg > 1 && c->g == c->Rg &&
        (int64_t)bytes * c->Rg > c->ll_max)
        return A_HIER;
    return A_PAIRWISE;
}

bool algo_valid(int op, int algo) {
    if (op == MPXA_OP_ALLTOALL) return algo == A_PAIRWISE || algo == A_BRUCK || algo == A_HIER;
    if (op == MPXA_OP_ALLTOALLV) return algo == A_PAIRWISE || algo == A_HIER || algo == A_BRUCK;
    if (op == MPXA_OP_ALLGATHER) return algo == A_PAIRWISE || algo == A_BRUCK || algo == A_RING || algo == A_HIER;
    return false;
}


int load_selector_file(mpxa_comm_t c, const char *path) {
    std::ifstream f(path);
    if (!f) return MPXA_ERR_ARG;
    std::vector<SelEntry> t;
    std::string line;
    while (std::getline(f, line)) {
        auto h = line.find('#');
        if (h != std::string::npos) line = line.substr(0, h);
        std::stringstream ss(line);
        std::vector<std::string> tok;
        for (std::string x; ss >> x;) tok.push_back(x);
        if (tok.empty()) continue;
        // "op p R max_bytes algo" (any GPU count / group) or "op p R G g max_bytes algo"
        if (tok.size() != 5 && tok.size() != 7) return MPXA_ERR_ARG;
        const bool full = tok.size() == 7;
        const std::string &op = tok[0], &algo = tok.back();
        SelEntry e{};
        char *endp = nullptr;
        e.p = (int)strtol(tok[1].c_str(), &endp, 10);
        e.R = (int)strtol(tok[2].c_str(), &endp, 10);
        e.G = full ? (int)strtol(tok[3].c_str(), &endp, 10) : -1;
        e.g = full ? (int)strtol(tok[4].c_str(), &endp, 10) : -1;
        const unsigned long long mb = strtoull(tok[full ? 5 : 3].c_str(), &endp, 10);
        e.op = op == "alltoall" ? 0 : op == "alltoallv" ? 1 : op == "allgather" ? 2 : -1;
        e.algo = algo == "pairwise" ? 1 : algo == "bruck" ? 2 : algo == "hier" ? 3 : algo == "ring" ? 4 : 0;
        e.max_bytes = mb;
        if (e.op < 0 || !algo_valid(e.op, e.algo)) return MPXA_ERR_ARG;
        t.push_back(e);
    }
    c->selector = t;
    return MPXA_SUCCESS;
}

}  // namespace mpxa_rt

extern "C" {

// ---- registry / selector -----------------------------------------------------------------
int mpxa_set_algorithm(mpxa_comm_t c, mpxa_op_t op, mpxa_algo_t a) {
    if (!c || op < 0 || op > 2) return MPXA_ERR_ARG;
    if (a != MPXA_ALGO_DEFAULT && !algo_valid(op, a)) return MPXA_ERR_ALGO;
    c->user_algo[op] = a;
    return MPXA_SUCCESS;
}

int mpxa_get_algorithm(mpxa_comm_t c, mpxa_op_t op, size_t bytes, mpxa_algo_t *chosen) {
    if (!c || !chosen || op < 0 || op > 2) return MPXA_ERR_ARG;
    *chosen = (mpxa_algo_t)default_algo(c, op, bytes);
    return MPXA_SUCCESS;
}

int mpxa_list_algorithms(mpxa_op_t op, mpxa_algo_t *out, int *n) {
    if (!n || op < 0 || op > 3) return MPXA_ERR_ARG;
    static const mpxa_algo_t a2a[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_BRUCK, MPXA_ALGO_HIER};
    static const mpxa_algo_t a2av[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_HIER, MPXA_ALGO_BRUCK};
    static const mpxa_algo_t ag[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_BRUCK, MPXA_ALGO_RING, MPXA_ALGO_HIER};
    static const mpxa_algo_t nb[] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_LOCALITY};
    const mpxa_algo_t *src = op == 0 ? a2a : op == 1 ? a2av : op == 2 ? ag : nb;
    int cnt = op == 3 ? 2 : op == 2 ? 4 : 3;
    if (out) {
        if (*n < cnt) { *n = cnt; return MPXA_ERR_ARG; }
        for (int i = 0; i < cnt; i++) out[i] = src[i];
    }
    *n = cnt;
    return MPXA_SUCCESS;
}

int mpxa_load_selector(mpxa_comm_t c, const char *path) {
    if (!c || !path) return MPXA_ERR_ARG;
    return load_selector_file(c, path);
}

int mpxa_config_digest(mpxa_comm_t c, uint64_t *digest) {
    if (!c || !digest) return MPXA_ERR_ARG;
    *digest = knob_digest(c, c->heap0);
    return MPXA_SUCCESS;
}

}  // extern "C"

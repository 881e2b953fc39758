/*
 * mpxa CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load or call this file.  The product path (paper_2309_07337_b200/) never
 * links, imports or executes it, and it shares no code with the product: no headers,
 * helpers, tables or generators.  Inputs come from the seeded generator module synth/.
 *
 * What it is: a plain, slow, single-threaded simulation of p MPI ranks exchanging
 * messages through an in-process transport with one FIFO per (src, dst) link and
 * message/byte counters ("transport").  Sends are
 * eager (buffered), so "every rank sends, then every rank receives" is a legal
 * execution of each round.  Every payload byte is moved with memcpy; nothing is
 * blocked, fused or reordered beyond what the algorithm states.
 *
 * Paper passages followed (PAPER.md = arXiv 2309.07337 LaTeX):
 *   - MPI_Alltoallv / MPIX_Alltoallv semantics, Listings 1-2, PAPER.md:104-118 (§2.1).
 *   - "minimize message count for small data sizes and bytes transported for larger
 *     messages" (Bruck vs pairwise) and "distinguishing between inter- and intra- node
 *     communication, reducing message count" (hierarchical), PAPER.md:98 (§2.1).
 *   - The paper gives no algorithm steps; the step lists are the ones BASELINE.json's
 *     north_star names ("local rotation, bit-indexed block send/recv, final inverse
 *     rotation"; "gather blocks within a group, exchange once between groups,
 *     redistribute") as read in SURVEY.md §8(c) C.4, items 1-7, and DESIGN.md §3.
 *
 * Pinning: tests/test_oracle_pins.py checks every function against numpy transposes /
 * concatenations, brute force with unique byte labels, closed-form message counts and
 * the Bruck per-round invariants.  No function here is "parity unpinned".
 *
 * Layout conventions (all buffers host memory, caller-owned):
 *   alltoall : send is p rows of p*blk bytes (row r = rank r, block j -> rank j),
 *              recv likewise (block j of row r came from rank j).
 *   allgather: send is p rows of blk bytes; recv is p rows of p*blk bytes.
 *   alltoallv: send rows of sstride bytes, recv rows of rstride bytes; counts and
 *              displacements are p*p int64 arrays in ELEMENTS of w bytes,
 *              sc[r*p+j] = sendcounts of rank r for destination j, rc[r*p+j] =
 *              recvcounts of rank r from source j (MPI semantics).
 * Return value: 0 on success, -1 on bad arguments, -2 on internal inconsistency
 * (a receive that found no matching message, which would be a deadlock in MPI).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* Statistics (SPEC.md:37-42 TransportStats; loopback messages are counted) */
typedef struct {
    int64_t ppn;          /* input: ranks per node for the intra/inter split (0 -> p)   */
    int64_t msgs;         /* total messages, including loopback                          */
    int64_t bytes;        /* total payload bytes                                          */
    int64_t intra_msgs, inter_msgs;
    int64_t intra_bytes, inter_bytes;
    int64_t max_msgs_per_rank;  /* max over ranks of messages sent                       */
    int64_t rounds;       /* communication rounds of the schedule                         */
} orc_stats;

/* ------------------------------------------------------------------------------------ */
/* Transport: one FIFO per (src, dst) link; matching on (src, dst, tag) in FIFO order.   */
typedef struct msg_s {
    int tag;
    size_t len;
    unsigned char *data;
    struct msg_s *next;
} msg_t;

typedef struct {
    int p;
    msg_t **head;   /* p*p FIFOs, index src*p+dst */
    msg_t **tail;
    int64_t *sent;  /* per-rank messages sent */
    orc_stats *st;
    int ppn;
} transport_t;

static int tp_init(transport_t *t, int p, orc_stats *st) {
    t->p = p;
    t->head = (msg_t **)calloc((size_t)p * p, sizeof(msg_t *));
    t->tail = (msg_t **)calloc((size_t)p * p, sizeof(msg_t *));
    t->sent = (int64_t *)calloc((size_t)p, sizeof(int64_t));
    t->st = st;
    t->ppn = (st && st->ppn > 0) ? (int)st->ppn : p;
    if (st) {
        int64_t keep = st->ppn;
        memset(st, 0, sizeof(*st));
        st->ppn = keep;
    }
    return (t->head && t->tail && t->sent) ? 0 : -1;
}

static int tp_pending(const transport_t *t) {
    for (int i = 0; i < t->p * t->p; i++)
        if (t->head[i]) return 1;
    return 0;
}

static void tp_free(transport_t *t) {
    for (int i = 0; i < t->p * t->p; i++) {
        msg_t *m = t->head[i];
        while (m) { msg_t *n = m->next; free(m->data); free(m); m = n; }
    }
    if (t->st) {
        int64_t mx = 0;
        for (int r = 0; r < t->p; r++) if (t->sent[r] > mx) mx = t->sent[r];
        t->st->max_msgs_per_rank = mx;
    }
    free(t->head); free(t->tail); free(t->sent);
}

/* eager send: the payload is copied into the envelope */
static int tp_send(transport_t *t, int src, int dst, int tag, const void *buf, size_t len) {
    msg_t *m = (msg_t *)malloc(sizeof(msg_t));
    if (!m) return -1;
    m->tag = tag; m->len = len; m->next = NULL;
    m->data = (unsigned char *)malloc(len ? len : 1);
    if (!m->data) { free(m); return -1; }
    if (len) memcpy(m->data, buf, len);
    int link = src * t->p + dst;
    if (t->tail[link]) t->tail[link]->next = m; else t->head[link] = m;
    t->tail[link] = m;
    t->sent[src]++;
    if (t->st) {
        int same = (src / t->ppn) == (dst / t->ppn);
        t->st->msgs++; t->st->bytes += (int64_t)len;
        if (same) { t->st->intra_msgs++; t->st->intra_bytes += (int64_t)len; }
        else      { t->st->inter_msgs++; t->st->inter_bytes += (int64_t)len; }
    }
    return 0;
}

/* blocking receive of the first message on link (src -> dst) with this tag.
 * Returns the payload length, or -1 if no such message exists (deadlock in MPI terms). */
static int64_t tp_recv(transport_t *t, int dst, int src, int tag, void *buf, size_t cap) {
    int link = src * t->p + dst;
    msg_t *prev = NULL, *m = t->head[link];
    while (m && m->tag != tag) { prev = m; m = m->next; }
    if (!m || m->len > cap) return -1;
    if (m->len) memcpy(buf, m->data, m->len);
    if (prev) prev->next = m->next; else t->head[link] = m->next;
    if (t->tail[link] == m) t->tail[link] = prev;
    int64_t n = (int64_t)m->len;
    free(m->data); free(m);
    return n;
}

static int imod(int64_t a, int p) { int64_t r = a % p; return (int)(r < 0 ? r + p : r); }
static int ceil_log2(int p) { int k = 0; while ((1 << k) < p) k++; return k; }

/* ==================================================================================== */
/* C.3 Definitions -- the result every variant must reach.                              */
/* ==================================================================================== */

/* alltoall identity recv_r[j] = send_j[r] (BASELINE.json north_star; MPI_Alltoall). */
int orc_alltoall_definition(int p, size_t blk, const unsigned char *send, unsigned char *recv) {
    if (p < 1) return -1;
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++)
            if (blk) memcpy(recv + ((size_t)r * p + j) * blk, send + ((size_t)j * p + r) * blk, blk);
    return 0;
}

/* allgather: recv_r[j] = send_j for all r (concatenation in rank order). */
int orc_allgather_definition(int p, size_t blk, const unsigned char *send, unsigned char *recv) {
    if (p < 1) return -1;
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++)
            if (blk) memcpy(recv + ((size_t)r * p + j) * blk, send + (size_t)j * blk, blk);
    return 0;
}

/* The same definition restricted to receiving ranks [r0, r1) -- so several host threads can
 * each fill their own receivers ("one thread per simulated rank");
 * the per-block copies are exactly orc_allgather_definition's. */
int orc_allgather_definition_rows(int p, size_t blk, const unsigned char *send, unsigned char *recv, int r0,
                                  int r1) {
    if (p < 1 || r0 < 0 || r1 > p || r0 > r1) return -1;
    for (int r = r0; r < r1; r++)
        for (int j = 0; j < p; j++)
            if (blk) memcpy(recv + ((size_t)r * p + j) * blk, send + (size_t)j * blk, blk);
    return 0;
}

/* Checks of the MPI alltoallv argument contract: non-negative counts,
 * in-bounds regions, sendcounts_j[r] == recvcounts_r[j]. */
static int v_args_ok(int p, size_t w, size_t sstride, const int64_t *sc, const int64_t *sd,
                     size_t rstride, const int64_t *rc, const int64_t *rd) {
    if (p < 1 || w < 1) return 0;
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++) {
            int64_t a = sc[r * p + j], b = sd[r * p + j], c = rc[r * p + j], d = rd[r * p + j];
            if (a < 0 || b < 0 || c < 0 || d < 0) return 0;
            if ((uint64_t)(b + a) * w > sstride) return 0;
            if ((uint64_t)(d + c) * w > rstride) return 0;
            if (sc[r * p + j] != rc[j * p + r]) return 0;
        }
    return 1;
}

/* alltoallv: recv_r[rd_r[j]*w, +rc_r[j]*w) = send_j[sd_j[r]*w, +sc_j[r]*w); all other bytes
 * of recv_r unchanged. */
int orc_alltoallv_definition(int p, size_t w, const unsigned char *send, size_t sstride,
                             const int64_t *sc, const int64_t *sd, unsigned char *recv,
                             size_t rstride, const int64_t *rc, const int64_t *rd) {
    if (!v_args_ok(p, w, sstride, sc, sd, rstride, rc, rd)) return -1;
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++) {
            size_t n = (size_t)rc[r * p + j] * w;
            if (n) memcpy(recv + (size_t)r * rstride + (size_t)rd[r * p + j] * w,
                          send + (size_t)j * sstride + (size_t)sd[j * p + r] * w, n);
        }
    return 0;
}

/* ==================================================================================== */
/* C.4 Variant simulations through the transport                                        */
/* ==================================================================================== */

/* C.4 item 1 -- pairwise alltoallv: for s = 0..p-1 every rank r sends its
 * segment for dst = (r+s) mod p and receives from src = (r-s) mod p; s = 0 is the
 * self-exchange (a loopback message).  p messages per rank, p^2 in total. */
int orc_alltoallv_pairwise(int p, size_t w, const unsigned char *send, size_t sstride,
                           const int64_t *sc, const int64_t *sd, unsigned char *recv,
                           size_t rstride, const int64_t *rc, const int64_t *rd, orc_stats *st) {
    if (!v_args_ok(p, w, sstride, sc, sd, rstride, rc, rd)) return -1;
    transport_t t;
    if (tp_init(&t, p, st)) return -1;
    int err = 0;
    for (int s = 0; s < p && !err; s++) {
        for (int r = 0; r < p && !err; r++) {
            int dst = imod(r + s, p);
            err = tp_send(&t, r, dst, s, send + (size_t)r * sstride + (size_t)sd[r * p + dst] * w,
                          (size_t)sc[r * p + dst] * w);
        }
        for (int r = 0; r < p && !err; r++) {
            int src = imod(r - s, p);
            int64_t n = tp_recv(&t, r, src, s, recv + (size_t)r * rstride + (size_t)rd[r * p + src] * w,
                                (size_t)rc[r * p + src] * w);
            if (n != rc[r * p + src] * (int64_t)w) err = -2;
        }
        if (st) st->rounds++;
    }
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    return err;
}

/* pairwise alltoall = pairwise alltoallv with every count = blk bytes, packed displs. */
int orc_alltoall_pairwise(int p, size_t blk, const unsigned char *send, unsigned char *recv,
                          orc_stats *st) {
    if (p < 1) return -1;
    int64_t *c = (int64_t *)malloc(sizeof(int64_t) * p * p);
    int64_t *d = (int64_t *)malloc(sizeof(int64_t) * p * p);
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++) { c[r * p + j] = (int64_t)blk; d[r * p + j] = (int64_t)blk * j; }
    int rc = orc_alltoallv_pairwise(p, 1, send, (size_t)p * blk, c, d, recv, (size_t)p * blk, c, d, st);
    free(c); free(d);
    return rc;
}

/* C.4 item 2 -- Bruck alltoall (BASELINE.json north_star: "local rotation, bit-indexed
 * block send/recv, final inverse rotation"; SURVEY.md Q1-Q3 conventions):
 *   R1  T_r[i] = send_r[(r+i) mod p]                                   (local rotation)
 *   R2  for k = 0..K-1, d = 2^k: rank r sends {T_r[i] : bit k of i is 1}, in increasing i,
 *       as ONE message to (r+d) mod p; the receiver stores the j-th received block at
 *       T[i_j] (same index set), i.e. it keeps the sender's pre-round values.
 *   R3  recv_r[j] = T_r[(r-j) mod p]                                   (inverse rotation)
 * stop_stage: -1 runs everything; 0 stops after R1; k+1 stops after round k.  When
 * T_out != NULL, T (p rows of p*blk) is copied there at the stop point (or at the end,
 * before R3, for stop_stage = -1). */
int orc_alltoall_bruck(int p, size_t blk, const unsigned char *send, unsigned char *recv,
                       int stop_stage, unsigned char *T_out, orc_stats *st) {
    if (p < 1) return -1;
    size_t row = (size_t)p * blk;
    unsigned char *T = (unsigned char *)malloc(row * p + 1);
    unsigned char *pack = (unsigned char *)malloc(row + 1);
    if (!T || !pack) { free(T); free(pack); return -1; }
    transport_t t;
    if (tp_init(&t, p, st)) { free(T); free(pack); return -1; }
    int err = 0;
    /* R1 */
    for (int r = 0; r < p; r++)
        for (int i = 0; i < p; i++)
            if (blk) memcpy(T + r * row + (size_t)i * blk, send + r * row + (size_t)imod(r + i, p) * blk, blk);
    int K = ceil_log2(p);
    int done = (stop_stage == 0);
    for (int k = 0; k < K && !done && !err; k++) {
        int d = 1 << k;
        for (int r = 0; r < p && !err; r++) {      /* every rank packs and sends */
            size_t n = 0;
            for (int i = 0; i < p; i++)
                if ((i >> k) & 1) { if (blk) memcpy(pack + n, T + r * row + (size_t)i * blk, blk); n += blk; }
            err = tp_send(&t, r, imod(r + d, p), k, pack, n);
        }
        for (int r = 0; r < p && !err; r++) {      /* every rank receives and unpacks */
            int src = imod(r - d, p);
            int64_t n = tp_recv(&t, r, src, k, pack, row);
            size_t o = 0;
            for (int i = 0; i < p; i++)
                if ((i >> k) & 1) { if (blk) memcpy(T + r * row + (size_t)i * blk, pack + o, blk); o += blk; }
            if (n != (int64_t)o) err = -2;
        }
        if (st) st->rounds++;
        if (stop_stage == k + 1) done = 1;
    }
    if (!err && T_out) memcpy(T_out, T, row * p);
    if (!err && !done)                               /* R3 */
        for (int r = 0; r < p; r++)
            for (int j = 0; j < p; j++)
                if (blk) memcpy(recv + r * row + (size_t)j * blk, T + r * row + (size_t)imod(r - j, p) * blk, blk);
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    free(T); free(pack);
    return err;
}

/* C.4 item 3 -- Bruck allgather: T_r[0] = send_r; for k = 0..K-1,
 * d = 2^k, n_k = min(d, p-d): rank r sends T_r[0..n_k) to (r-d) mod p, which stores them
 * at T[d..d+n_k); finally recv_r[j] = T_r[(j-r) mod p].  stop_stage as for alltoall
 * (0 = after T_r[0] = send_r). */
int orc_allgather_bruck(int p, size_t blk, const unsigned char *send, unsigned char *recv,
                        int stop_stage, unsigned char *T_out, orc_stats *st) {
    if (p < 1) return -1;
    size_t row = (size_t)p * blk;
    unsigned char *T = (unsigned char *)calloc(row * p + 1, 1);
    if (!T) return -1;
    transport_t t;
    if (tp_init(&t, p, st)) { free(T); return -1; }
    int err = 0;
    for (int r = 0; r < p; r++) if (blk) memcpy(T + r * row, send + (size_t)r * blk, blk);
    int K = ceil_log2(p);
    int done = (stop_stage == 0);
    for (int k = 0; k < K && !done && !err; k++) {
        int d = 1 << k, nk = d < p - d ? d : p - d;
        for (int r = 0; r < p && !err; r++)
            err = tp_send(&t, r, imod(r - d, p), k, T + r * row, (size_t)nk * blk);
        for (int r = 0; r < p && !err; r++) {
            int64_t n = tp_recv(&t, r, imod(r + d, p), k, T + r * row + (size_t)d * blk, (size_t)nk * blk);
            if (n != (int64_t)((size_t)nk * blk)) err = -2;
        }
        if (st) st->rounds++;
        if (stop_stage == k + 1) done = 1;
    }
    if (!err && T_out) memcpy(T_out, T, row * p);
    if (!err && !done)
        for (int r = 0; r < p; r++)
            for (int j = 0; j < p; j++)
                if (blk) memcpy(recv + r * row + (size_t)j * blk, T + r * row + (size_t)imod(j - r, p) * blk, blk);
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    free(T);
    return err;
}

/* C.4 item 4 -- ring allgather: recv_r[r] = send_r; for s = 0..p-2, rank r
 * sends block (r-s) mod p to (r+1) mod p, which stores it at index (r-s) mod p. */
int orc_allgather_ring(int p, size_t blk, const unsigned char *send, unsigned char *recv,
                       orc_stats *st) {
    if (p < 1) return -1;
    size_t row = (size_t)p * blk;
    transport_t t;
    if (tp_init(&t, p, st)) return -1;
    int err = 0;
    for (int r = 0; r < p; r++) if (blk) memcpy(recv + r * row + (size_t)r * blk, send + (size_t)r * blk, blk);
    for (int s = 0; s < p - 1 && !err; s++) {
        for (int r = 0; r < p && !err; r++) {
            int b = imod(r - s, p);
            err = tp_send(&t, r, imod(r + 1, p), s, recv + r * row + (size_t)b * blk, blk);
        }
        for (int r = 0; r < p && !err; r++) {
            int src = imod(r - 1, p), b = imod(src - s, p);
            int64_t n = tp_recv(&t, r, src, s, recv + r * row + (size_t)b * blk, blk);
            if (n != (int64_t)blk) err = -2;
        }
        if (st) st->rounds++;
    }
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    return err;
}

/* C.4 item 5 -- direct ("pairwise") allgather: r sends send_r to every j != r, and
 * copies it locally into recv_r[r]. */
int orc_allgather_direct(int p, size_t blk, const unsigned char *send, unsigned char *recv,
                         orc_stats *st) {
    if (p < 1) return -1;
    size_t row = (size_t)p * blk;
    transport_t t;
    if (tp_init(&t, p, st)) return -1;
    int err = 0;
    for (int r = 0; r < p; r++) if (blk) memcpy(recv + r * row + (size_t)r * blk, send + (size_t)r * blk, blk);
    for (int s = 1; s < p && !err; s++)
        for (int r = 0; r < p && !err; r++)
            err = tp_send(&t, r, imod(r + s, p), 0, send + (size_t)r * blk, blk);
    for (int s = 1; s < p && !err; s++)
        for (int r = 0; r < p && !err; r++) {
            int src = imod(r - s, p);
            int64_t n = tp_recv(&t, r, src, 0, recv + r * row + (size_t)src * blk, blk);
            if (n != (int64_t)blk) err = -2;
        }
    if (st) st->rounds = p > 1 ? 1 : 0;
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    return err;
}

/* C.4 item 6 -- locality-aware hierarchical alltoallv ("distinguishing between
 * inter- and intra- node communication, reducing message count"; SPEC.md:158-166, 220;
 * BASELINE.json north_star "gather blocks within a group, exchange once between groups,
 * redistribute").  Groups are contiguous of size g; group of r is A = r/g;
 * leader L(A,B) = A*g + (B mod g).
 *   Step 1: every rank r in A, for every remote group B, sends ONE message to L(A,B) with
 *           its g segments (r -> B*g+t), t = 0..g-1, concatenated in t order.
 *   Step 2: L(A,B) sends L(B,A) ONE aggregated message with segments ordered (s,t)
 *           row-major (s = source local index in A, t = destination local index in B);
 *           empty group pairs send no message.
 *   Step 3: L(B,A) sends each rank B*g+t ONE message with its g segments (s = 0..g-1);
 *           the rank stores segment s at rdispls[A*g+s].
 *   Intra-group pairs (B = A) are exchanged directly.
 * The aggregated layout is fixed by the count matrix (no in-band headers).
 * st->ppn should be set to g by the caller to count inter-group messages. */
int orc_alltoallv_hier(int p, int g, size_t w, const unsigned char *send, size_t sstride,
                       const int64_t *sc, const int64_t *sd, unsigned char *recv, size_t rstride,
                       const int64_t *rc, const int64_t *rd, orc_stats *st) {
    if (g < 1 || p % g) return -1;
    if (!v_args_ok(p, w, sstride, sc, sd, rstride, rc, rd)) return -1;
    int G = p / g;
    transport_t t;
    if (tp_init(&t, p, st)) return -1;
    int err = 0;
    size_t cap = 0;   /* largest message any step can carry */
    for (int a = 0; a < p; a++)
        for (int b = 0; b < p; b++) cap += (size_t)sc[a * p + b] * w;
    unsigned char *buf = (unsigned char *)malloc(cap + 1);
    unsigned char *agg = (unsigned char *)malloc(cap + 1);
    if (!buf || !agg) { free(buf); free(agg); tp_free(&t); return -1; }
    enum { TAG_DIRECT = 1, TAG_GATHER = 2, TAG_EXCH = 3, TAG_SCATTER = 4 };

    /* intra-group direct exchange */
    for (int r = 0; r < p && !err; r++) {
        int A = r / g;
        for (int u = 0; u < g && !err; u++) {
            int j = A * g + u;
            err = tp_send(&t, r, j, TAG_DIRECT, send + (size_t)r * sstride + (size_t)sd[r * p + j] * w,
                          (size_t)sc[r * p + j] * w);
        }
    }
    for (int r = 0; r < p && !err; r++) {
        int A = r / g;
        for (int u = 0; u < g && !err; u++) {
            int j = A * g + u;
            int64_t n = tp_recv(&t, r, j, TAG_DIRECT, recv + (size_t)r * rstride + (size_t)rd[r * p + j] * w,
                                (size_t)rc[r * p + j] * w);
            if (n != rc[r * p + j] * (int64_t)w) err = -2;
        }
    }
    /* Step 1: gather to L(A,B) */
    for (int r = 0; r < p && !err; r++) {
        int A = r / g;
        for (int B = 0; B < G && !err; B++) {
            if (B == A) continue;
            size_t n = 0;
            for (int u = 0; u < g; u++) {
                int j = B * g + u;
                size_t len = (size_t)sc[r * p + j] * w;
                if (len) memcpy(buf + n, send + (size_t)r * sstride + (size_t)sd[r * p + j] * w, len);
                n += len;
            }
            err = tp_send(&t, r, A * g + (B % g), TAG_GATHER + 8 * B, buf, n);
        }
    }
    if (st && G > 1) st->rounds++;
    /* Step 2: each leader L(A,B) receives the g gathered messages, lays them out (s,t)
     * row-major, and sends one aggregated message to L(B,A) */
    for (int A = 0; A < G && !err; A++)
        for (int B = 0; B < G && !err; B++) {
            if (B == A) continue;
            int lead = A * g + (B % g), peer = B * g + (A % g);
            size_t n = 0;
            for (int s = 0; s < g && !err; s++) {
                int src = A * g + s;
                size_t want = 0;
                for (int u = 0; u < g; u++) want += (size_t)sc[src * p + B * g + u] * w;
                int64_t got = tp_recv(&t, lead, src, TAG_GATHER + 8 * B, agg + n, cap - n);
                if (got != (int64_t)want) err = -2;
                n += want;
            }
            if (!err && n) err = tp_send(&t, lead, peer, TAG_EXCH + 8 * A, agg, n);
        }
    if (st && G > 1) st->rounds++;
    /* Step 3: L(B,A) receives from L(A,B) and redistributes segment (s,t) to B*g+t */
    for (int B = 0; B < G && !err; B++)
        for (int A = 0; A < G && !err; A++) {
            if (A == B) continue;
            int lead = B * g + (A % g), peer = A * g + (B % g);
            size_t total = 0;
            for (int s = 0; s < g; s++)
                for (int u = 0; u < g; u++) total += (size_t)sc[(A * g + s) * p + B * g + u] * w;
            if (total) {
                int64_t got = tp_recv(&t, lead, peer, TAG_EXCH + 8 * A, agg, cap);
                if (got != (int64_t)total) { err = -2; break; }
            }
            for (int u = 0; u < g && !err; u++) {
                size_t n = 0;
                for (int s = 0; s < g; s++) {      /* segment (s,u) offset in (s,t) row-major */
                    size_t off = 0;
                    for (int s2 = 0; s2 < g; s2++)
                        for (int u2 = 0; u2 < g; u2++) {
                            if (s2 == s && u2 == u) goto found;
                            off += (size_t)sc[(A * g + s2) * p + B * g + u2] * w;
                        }
                found:;
                    size_t len = (size_t)sc[(A * g + s) * p + B * g + u] * w;
                    if (len) memcpy(buf + n, agg + off, len);
                    n += len;
                }
                err = tp_send(&t, lead, B * g + u, TAG_SCATTER + 8 * A, buf, n);
            }
        }
    if (st && G > 1) st->rounds++;
    for (int r = 0; r < p && !err; r++) {
        int B = r / g, u = r % g;
        for (int A = 0; A < G && !err; A++) {
            if (A == B) continue;
            int lead = B * g + (A % g);
            size_t want = 0;
            for (int s = 0; s < g; s++) want += (size_t)rc[r * p + A * g + s] * w;
            int64_t got = tp_recv(&t, r, lead, TAG_SCATTER + 8 * A, buf, cap);
            if (got != (int64_t)want) { err = -2; break; }
            size_t o = 0;
            for (int s = 0; s < g; s++) {
                size_t len = (size_t)rc[r * p + A * g + s] * w;
                if (len) memcpy(recv + (size_t)r * rstride + (size_t)rd[r * p + A * g + s] * w, buf + o, len);
                o += len;
            }
        }
        (void)u;
    }
    if (!err && tp_pending(&t)) err = -2;
    free(buf); free(agg);
    tp_free(&t);
    return err;
}

/* hierarchical alltoall = hierarchical alltoallv with uniform counts. */
int orc_alltoall_hier(int p, int g, size_t blk, const unsigned char *send, unsigned char *recv,
                      orc_stats *st) {
    if (p < 1) return -1;
    int64_t *c = (int64_t *)malloc(sizeof(int64_t) * p * p);
    int64_t *d = (int64_t *)malloc(sizeof(int64_t) * p * p);
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++) { c[r * p + j] = (int64_t)blk; d[r * p + j] = (int64_t)blk * j; }
    int rc = orc_alltoallv_hier(p, g, 1, send, (size_t)p * blk, c, d, recv, (size_t)p * blk, c, d, st);
    free(c); free(d);
    return rc;
}

/* C.4 item 7 -- counts exchange + displacement scan (BASELINE.json cfg4 "counts/displs
 * exchanged then data"): recvcounts = alltoall of sendcounts (one int64 per pair, sent as
 * messages through the transport); rdispls_r[j] = sum_{i<j} recvcounts_r[i]. */
int orc_counts_exchange(int p, const int64_t *sendcounts, int64_t *recvcounts, int64_t *rdispls,
                        orc_stats *st) {
    if (p < 1) return -1;
    transport_t t;
    if (tp_init(&t, p, st)) return -1;
    int err = 0;
    for (int s = 0; s < p && !err; s++) {
        for (int r = 0; r < p && !err; r++) {
            int dst = imod(r + s, p);
            err = tp_send(&t, r, dst, 0, &sendcounts[r * p + dst], sizeof(int64_t));
        }
        for (int r = 0; r < p && !err; r++) {
            int src = imod(r - s, p);
            if (tp_recv(&t, r, src, 0, &recvcounts[r * p + src], sizeof(int64_t)) != (int64_t)sizeof(int64_t)) err = -2;
        }
    }
    for (int r = 0; r < p && !err; r++) {
        int64_t acc = 0;
        for (int j = 0; j < p; j++) { rdispls[r * p + j] = acc; acc += recvcounts[r * p + j]; }
    }
    tp_free(&t);
    return err;
}

/* ==================================================================================== */
/* f1: persistent neighborhood alltoallv (§2.2).      */
/*                                                                                      */
/* Graph layout (global view, one entry list per rank, rank-major):                     */
/*   indeg[r], and for r's in-edges k (in order): src, rc (count, elements), rd (displ)  */
/*   outdeg[r], and for r's out-edges k: dst, sc, sd.                                    */
/* Edges are matched like MPI matches messages: the j-th out-edge of r towards q pairs   */
/* with the j-th in-edge of q from r (multigraphs allowed); counts must agree.           */
/* Locality variant: send_idx / recv_idx hold one global index per element, laid out     */
/* edge by edge in edge order (r's out-edges: sc[k] ids each; q's in-edges likewise).     */
/* ==================================================================================== */

/* position of the out-edge of r that pairs with in-edge kin of q (-1 if none) */
static int64_t nb_match(const int *outdeg, const int64_t *ooff, const int *dst,
                        const int *indeg, const int64_t *ioff, const int *src, int q, int kin) {
    int r = src[ioff[q] + kin];
    int occ = 0;
    for (int k = 0; k < kin; k++) if (src[ioff[q] + k] == r) occ++;
    for (int k = 0; k < outdeg[r]; k++)
        if (dst[ooff[r] + k] == q) {
            if (occ == 0) return ooff[r] + k;
            occ--;
        }
    (void)indeg;
    return -1;
}

static void nb_offsets(int p, const int *deg, int64_t *off) {
    off[0] = 0;
    for (int r = 0; r < p; r++) off[r + 1] = off[r] + deg[r];
}

/* Checks of the Dist_graph / Neighbor_alltoallv contract:
 * valid ranks, non-negative counts, in-bounds regions, every in-edge matched by an
 * out-edge of the same count and every out-edge matched. */
static int nb_args_ok(int p, size_t w, const int *indeg, const int *src, const int64_t *rc,
                      const int64_t *rd, size_t rstride, const int *outdeg, const int *dst,
                      const int64_t *sc, const int64_t *sd, size_t sstride, int64_t *ioff,
                      int64_t *ooff) {
    if (p < 1 || w < 1) return 0;
    nb_offsets(p, indeg, ioff);
    nb_offsets(p, outdeg, ooff);
    for (int r = 0; r < p; r++) {
        if (indeg[r] < 0 || outdeg[r] < 0) return 0;
        for (int64_t e = ioff[r]; e < ioff[r + 1]; e++) {
            if (src[e] < 0 || src[e] >= p || rc[e] < 0 || rd[e] < 0) return 0;
            if ((uint64_t)(rc[e] + rd[e]) * w > rstride) return 0;
        }
        for (int64_t e = ooff[r]; e < ooff[r + 1]; e++) {
            if (dst[e] < 0 || dst[e] >= p || sc[e] < 0 || sd[e] < 0) return 0;
            if ((uint64_t)(sc[e] + sd[e]) * w > sstride) return 0;
        }
    }
    int64_t nin = ioff[p], matched = 0;
    for (int q = 0; q < p; q++)
        for (int k = 0; k < indeg[q]; k++) {
            int64_t o = nb_match(outdeg, ooff, dst, indeg, ioff, src, q, k);
            if (o < 0 || sc[o] != rc[ioff[q] + k]) return 0;
            matched++;
        }
    return matched == nin && nin == ooff[p];
}

/* Definition (MPI_Neighbor_alltoallv, Listing 3): for every in-edge k of q
 * from r, recv_q[rd*w, +rc*w) = the bytes r's matching out-edge names in send_r; every other
 * byte of recv_q unchanged. */
int orc_neighbor_definition(int p, size_t w, const int *indeg, const int *src, const int64_t *rc,
                            const int64_t *rd, unsigned char *recv, size_t rstride, const int *outdeg,
                            const int *dst, const int64_t *sc, const int64_t *sd,
                            const unsigned char *send, size_t sstride) {
    int64_t *ioff = (int64_t *)malloc(sizeof(int64_t) * (p + 1));
    int64_t *ooff = (int64_t *)malloc(sizeof(int64_t) * (p + 1));
    int ok = nb_args_ok(p, w, indeg, src, rc, rd, rstride, outdeg, dst, sc, sd, sstride, ioff, ooff);
    if (ok)
        for (int q = 0; q < p; q++)
            for (int k = 0; k < indeg[q]; k++) {
                int64_t e = ioff[q] + k, o = nb_match(outdeg, ooff, dst, indeg, ioff, src, q, k);
                if (rc[e])
                    memcpy(recv + (size_t)q * rstride + (size_t)rd[e] * w,
                           send + (size_t)src[e] * sstride + (size_t)sd[o] * w, (size_t)rc[e] * w);
            }
    free(ioff); free(ooff);
    return ok ? 0 : -1;
}

/* Standard persistent neighbor alltoallv: one message per out-edge with
 * count > 0 (tag = occurrence of that destination among the rank's out-edges), then every
 * rank receives its in-edges in order.  Counters: msgs = edges with count > 0. */
int orc_neighbor_standard(int p, size_t w, const int *indeg, const int *src, const int64_t *rc,
                          const int64_t *rd, unsigned char *recv, size_t rstride, const int *outdeg,
                          const int *dst, const int64_t *sc, const int64_t *sd,
                          const unsigned char *send, size_t sstride, orc_stats *st) {
    int64_t *ioff = (int64_t *)malloc(sizeof(int64_t) * (p + 1));
    int64_t *ooff = (int64_t *)malloc(sizeof(int64_t) * (p + 1));
    int err = nb_args_ok(p, w, indeg, src, rc, rd, rstride, outdeg, dst, sc, sd, sstride, ioff, ooff) ? 0 : -1;
    transport_t t;
    if (!err && tp_init(&t, p, st)) err = -1;
    if (!err) {
        for (int r = 0; r < p && !err; r++)
            for (int k = 0; k < outdeg[r] && !err; k++) {
                int64_t e = ooff[r] + k;
                int occ = 0;
                for (int k2 = 0; k2 < k; k2++) if (dst[ooff[r] + k2] == dst[e]) occ++;
                if (sc[e]) err = tp_send(&t, r, dst[e], occ, send + (size_t)r * sstride + (size_t)sd[e] * w,
                                         (size_t)sc[e] * w);
            }
        if (st) st->rounds = 1;
        for (int q = 0; q < p && !err; q++)
            for (int k = 0; k < indeg[q] && !err; k++) {
                int64_t e = ioff[q] + k;
                int occ = 0;
                for (int k2 = 0; k2 < k; k2++) if (src[ioff[q] + k2] == src[e]) occ++;
                if (rc[e] && tp_recv(&t, q, src[e], occ, recv + (size_t)q * rstride + (size_t)rd[e] * w,
                                     (size_t)rc[e] * w) != rc[e] * (int64_t)w) err = -2;
            }
        if (!err && tp_pending(&t)) err = -2;
        tp_free(&t);
    }
    free(ioff); free(ooff);
    return err;
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : x > y;
}

/* sorted unique copy of v[0..n) into out; returns the count */
static int64_t uniq_sorted(const int64_t *v, int64_t n, int64_t *out) {
    if (n <= 0) return 0;
    memcpy(out, v, sizeof(int64_t) * (size_t)n);
    qsort(out, (size_t)n, sizeof(int64_t), cmp_i64);
    int64_t m = 1;
    for (int64_t i = 1; i < n; i++) if (out[i] != out[m - 1]) out[m++] = out[i];
    return m;
}

static int64_t find_sorted(const int64_t *v, int64_t n, int64_t x) {
    int64_t lo = 0, hi = n - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (v[mid] == x) return mid;
        if (v[mid] < x) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

#define NB_TAG_FWD 100000
#define NB_TAG_EXCH 200000
#define NB_TAG_FAN 300000

/* Locality-aware persistent neighbor alltoallv with unique value indices (PAPER.md:157:
 * "unique indices for all values ... eliminate a single value from being sent between a set
 * of nodes multiple times"; three-phase plan of SPEC.md:307-315).  Nodes are groups of g
 * consecutive ranks; the aggregator for (node A, remote node B) is leader_for(B) on A =
 * A*g + (B mod g).  Messages carry (index, value) records, index sorted:
 *   (1) every rank r of A sends, per remote node B, the set of unique indices among its
 *       elements bound for ranks of B (per-sender dedup), with their values, to L(A,B);
 *   (2) L(A,B) merges the sets of its node's senders (one record per index) and sends ONE
 *       message with each unique index once to L(B,A);
 *   (3) L(B,A) sends every rank q of B the values of its in-edge elements from node A, in
 *       q's element order; q stores them at its receive displacements.
 * Intra-node edges are sent directly (standard).  *inter_values counts the (index,value)
 * records crossing node boundaries (phase 2).  Returns -3 when a received element's index
 * differs from the index of the element its edge matches (inconsistent recv_indices). */
int orc_neighbor_locality(int p, int g, size_t w, const int *indeg, const int *src, const int64_t *rc,
                          const int64_t *rd, const int64_t *recv_idx, unsigned char *recv, size_t rstride,
                          const int *outdeg, const int *dst, const int64_t *sc, const int64_t *sd,
                          const int64_t *send_idx, const unsigned char *send, size_t sstride, orc_stats *st,
                          int64_t *inter_values) {
    if (g < 1 || p % g) return -1;
    int64_t *ioff = (int64_t *)malloc(sizeof(int64_t) * (p + 1));
    int64_t *ooff = (int64_t *)malloc(sizeof(int64_t) * (p + 1));
    int err = nb_args_ok(p, w, indeg, src, rc, rd, rstride, outdeg, dst, sc, sd, sstride, ioff, ooff) ? 0 : -1;
    if (err) { free(ioff); free(ooff); return err; }
    const int G = p / g;
    /* element offsets of every edge in the index arrays */
    int64_t *oe = (int64_t *)malloc(sizeof(int64_t) * (ooff[p] + 1));
    int64_t *ie = (int64_t *)malloc(sizeof(int64_t) * (ioff[p] + 1));
    oe[0] = 0; for (int64_t e = 0; e < ooff[p]; e++) oe[e + 1] = oe[e] + sc[e];
    ie[0] = 0; for (int64_t e = 0; e < ioff[p]; e++) ie[e + 1] = ie[e] + rc[e];
    /* consistency handshake: each received element's index equals its matched sent index */
    for (int q = 0; q < p && !err; q++)
        for (int k = 0; k < indeg[q] && !err; k++) {
            int64_t e = ioff[q] + k, o = nb_match(outdeg, ooff, dst, indeg, ioff, src, q, k);
            for (int64_t x = 0; x < rc[e]; x++)
                if (recv_idx[ie[e] + x] != send_idx[oe[o] + x]) { err = -3; break; }
        }
    int64_t nel = oe[ooff[p]] + ie[ioff[p]] + 1;
    size_t rec = sizeof(int64_t) + w;                     /* (index, value) record */
    int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)nel);
    int64_t *uq = (int64_t *)malloc(sizeof(int64_t) * (size_t)nel);
    unsigned char *buf = (unsigned char *)malloc(rec * (size_t)nel);
    unsigned char *agg = (unsigned char *)malloc(rec * (size_t)nel);
    transport_t t;
    if (!err && tp_init(&t, p, st)) err = -1;
    if (err) goto out_noT;
    if (inter_values) *inter_values = 0;
    /* intra-node edges: direct (standard) messages */
    for (int r = 0; r < p && !err; r++)
        for (int k = 0; k < outdeg[r] && !err; k++) {
            int64_t e = ooff[r] + k;
            if (dst[e] / g != r / g || !sc[e]) continue;
            int occ = 0;
            for (int k2 = 0; k2 < k; k2++) if (dst[ooff[r] + k2] == dst[e]) occ++;
            err = tp_send(&t, r, dst[e], occ, send + (size_t)r * sstride + (size_t)sd[e] * w, (size_t)sc[e] * w);
        }
    /* phase 1: per-sender dedup, forward (index, value) records to L(A,B) */
    for (int r = 0; r < p && !err; r++) {
        int A = r / g;
        for (int B = 0; B < G && !err; B++) {
            if (B == A) continue;
            int64_t n = 0;
            for (int k = 0; k < outdeg[r]; k++) {
                int64_t e = ooff[r] + k;
                if (dst[e] / g == B) for (int64_t x = 0; x < sc[e]; x++) ids[n++] = send_idx[oe[e] + x];
            }
            int64_t m = uniq_sorted(ids, n, uq);
            /* value of each unique index: its first element in (edge, element) order */
            int64_t *first = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
            for (int64_t u = 0; u < m; u++) first[u] = -1;
            for (int k = 0; k < outdeg[r]; k++) {
                int64_t e = ooff[r] + k;
                if (dst[e] / g != B) continue;
                for (int64_t x = 0; x < sc[e]; x++) {
                    int64_t u = find_sorted(uq, m, send_idx[oe[e] + x]);
                    if (first[u] < 0) first[u] = sd[e] + x;        /* element offset in send_r */
                }
            }
            for (int64_t u = 0; u < m; u++) {
                memcpy(buf + rec * u, &uq[u], sizeof(int64_t));
                memcpy(buf + rec * u + sizeof(int64_t), send + (size_t)r * sstride + (size_t)first[u] * w, w);
            }
            free(first);
            if (m) err = tp_send(&t, r, A * g + (B % g), NB_TAG_FWD + B, buf, rec * (size_t)m);
        }
    }
    if (st) st->rounds++;
    /* phase 2: L(A,B) merges its node's records (one per index) and sends one message */
    for (int A = 0; A < G && !err; A++)
        for (int B = 0; B < G && !err; B++) {
            if (B == A) continue;
            int lead = A * g + (B % g), peer = B * g + (A % g);
            int64_t n = 0;
            for (int s = 0; s < g && !err; s++) {
                int64_t got = tp_recv(&t, lead, A * g + s, NB_TAG_FWD + B, agg + rec * n, rec * (size_t)(nel - n));
                if (got == -1) continue;                       /* that sender had nothing for B */
                n += got / (int64_t)rec;
            }
            /* merge: one record per index (the first received), index ascending */
            for (int64_t i = 0; i < n; i++) memcpy(&ids[i], agg + rec * i, sizeof(int64_t));
            int64_t m = uniq_sorted(ids, n, uq);
            int64_t *first = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
            for (int64_t u = 0; u < m; u++) first[u] = -1;
            for (int64_t i = 0; i < n; i++) {
                int64_t u = find_sorted(uq, m, ids[i]);
                if (first[u] < 0) first[u] = i;
            }
            for (int64_t u = 0; u < m; u++) memcpy(buf + rec * u, agg + rec * first[u], rec);
            free(first);
            if (m) {
                err = tp_send(&t, lead, peer, NB_TAG_EXCH + A, buf, rec * (size_t)m);
                if (inter_values) *inter_values += m;
            }
        }
    if (st) st->rounds++;
    /* phase 3: L(B,A) fans the values out to every rank q of B, in q's element order */
    for (int B = 0; B < G && !err; B++)
        for (int A = 0; A < G && !err; A++) {
            if (A == B) continue;
            int lead = B * g + (A % g), peer = A * g + (B % g);
            int64_t got = tp_recv(&t, lead, peer, NB_TAG_EXCH + A, agg, rec * (size_t)nel);
            int64_t m = got < 0 ? 0 : got / (int64_t)rec;
            for (int64_t u = 0; u < m; u++) memcpy(&uq[u], agg + rec * u, sizeof(int64_t));
            for (int qq = 0; qq < g && !err; qq++) {
                int q = B * g + qq;
                int64_t n = 0;
                for (int k = 0; k < indeg[q] && !err; k++) {
                    int64_t e = ioff[q] + k;
                    if (src[e] / g != A) continue;
                    for (int64_t x = 0; x < rc[e]; x++) {
                        int64_t u = find_sorted(uq, m, recv_idx[ie[e] + x]);
                        if (u < 0) { err = -2; break; }
                        memcpy(buf + w * n, agg + rec * u + sizeof(int64_t), w);
                        n++;
                    }
                }
                if (!err && n) err = tp_send(&t, lead, q, NB_TAG_FAN + A, buf, w * (size_t)n);
            }
        }
    if (st) st->rounds++;
    /* receivers: direct intra-node edges, then one fan-out message per remote node */
    for (int q = 0; q < p && !err; q++) {
        int B = q / g;
        for (int k = 0; k < indeg[q] && !err; k++) {
            int64_t e = ioff[q] + k;
            if (src[e] / g != B || !rc[e]) continue;
            int occ = 0;
            for (int k2 = 0; k2 < k; k2++) if (src[ioff[q] + k2] == src[e]) occ++;
            if (tp_recv(&t, q, src[e], occ, recv + (size_t)q * rstride + (size_t)rd[e] * w, (size_t)rc[e] * w) !=
                rc[e] * (int64_t)w) err = -2;
        }
        for (int A = 0; A < G && !err; A++) {
            if (A == B) continue;
            int64_t need = 0;
            for (int k = 0; k < indeg[q]; k++) if (src[ioff[q] + k] / g == A) need += rc[ioff[q] + k];
            if (!need) continue;
            if (tp_recv(&t, q, B * g + (A % g), NB_TAG_FAN + A, buf, w * (size_t)nel) != need * (int64_t)w) {
                err = -2;
                break;
            }
            int64_t n = 0;
            for (int k = 0; k < indeg[q]; k++) {
                int64_t e = ioff[q] + k;
                if (src[e] / g != A) continue;
                if (rc[e]) memcpy(recv + (size_t)q * rstride + (size_t)rd[e] * w, buf + w * n, (size_t)rc[e] * w);
                n += rc[e];
            }
        }
    }
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
out_noT:
    free(ids); free(uq); free(buf); free(agg); free(oe); free(ie); free(ioff); free(ooff);
    return err;
}

/* ==================================================================================== */
/* f3: partitioned point-to-point (§2.3).              */
/* A channel moves one message of n_s * bs bytes; the sender marks n_s equal partitions   */
/* ready (Pready), the receiver sees n_r equal partitions of br bytes (same total) and   */
/* asks whether each has arrived (Parrived): "partitions of the same or different sizes  */
/* can be accessed as complete, prior to completion of the whole message". */
/* ==================================================================================== */

/* Parrived by byte coverage ("arrived(i) iff the byte interval of receiver
 * partition i is fully covered by delivered fragments"): brute force over bytes. */
int orc_part_arrived(int n_s, size_t bs, int n_r, size_t br, const unsigned char *delivered,
                     unsigned char *arrived) {
    if (n_s < 1 || n_r < 1 || (size_t)n_s * bs != (size_t)n_r * br) return -1;
    for (int j = 0; j < n_r; j++) {
        int ok = 1;
        for (size_t b = (size_t)j * br; b < (size_t)(j + 1) * br && ok; b++)
            if (!delivered[b / (bs ? bs : 1)]) ok = 0;
        arrived[j] = (unsigned char)ok;
    }
    return 0;
}

/* One cycle through the transport: the sender readies partitions in `order` (a permutation
 * of 0..n_s-1); each Pready sends one fragment (partition bytes; tag = partition index)
 * that the receiver integrates on arrival (one fragment per READY
 * partition).  After the k-th delivery, arrived_trace[k*n_r + j] = Parrived(j).  Returns
 * the receiver buffer in recv; stats count fragments (messages). */
int orc_part_cycle(int n_s, size_t bs, int n_r, size_t br, const unsigned char *send, unsigned char *recv,
                   const int *order, unsigned char *arrived_trace, orc_stats *st) {
    if (n_s < 1 || n_r < 1 || (size_t)n_s * bs != (size_t)n_r * br) return -1;
    transport_t t;
    if (tp_init(&t, 2, st)) return -1;
    unsigned char *delivered = (unsigned char *)calloc((size_t)n_s, 1);
    int err = 0;
    for (int k = 0; k < n_s && !err; k++) {
        int i = order[k];
        if (i < 0 || i >= n_s || delivered[i]) { err = -1; break; }
        err = tp_send(&t, 0, 1, i, send + (size_t)i * bs, bs);            /* Pready(i) */
        if (!err && tp_recv(&t, 1, 0, i, recv + (size_t)i * bs, bs) != (int64_t)bs) err = -2;
        delivered[i] = 1;
        if (!err) err = orc_part_arrived(n_s, bs, n_r, br, delivered, arrived_trace + (size_t)k * n_r);
    }
    if (st) st->rounds = n_s;
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    free(delivered);
    return err;
}

/* f2(i): hierarchical allgather ("intra-node gather to leader, inter-node bruck
 * among leaders, intra-node broadcast"; the locality-aware allgather family PAPER.md:173 cites).
 * Nodes are groups of g consecutive ranks with leader A*g.  (1) every rank sends its block to
 * its leader; (2) the G leaders run the Bruck allgather (C.4 item 3) on their node aggregates
 * of g blocks; (3) every leader sends the full p-block result to each of its other ranks. */
int orc_allgather_hier(int p, int g, size_t blk, const unsigned char *send, unsigned char *recv, orc_stats *st) {
    if (p < 1 || g < 1 || p % g) return -1;
    const int G = p / g, K = ceil_log2(G);
    const size_t agg = (size_t)g * blk;
    transport_t t;
    if (tp_init(&t, p, st)) return -1;
    unsigned char *T = (unsigned char *)calloc((size_t)G * (size_t)p * blk + 1, 1);   /* per leader: G aggregates */
    unsigned char *buf = (unsigned char *)malloc((size_t)p * blk + 1);
    int err = 0;
    /* (1) gather to the node leader (self included, as a loopback message) */
    for (int r = 0; r < p && !err; r++) err = tp_send(&t, r, (r / g) * g, 1, send + (size_t)r * blk, blk);
    for (int A = 0; A < G && !err; A++)
        for (int s = 0; s < g && !err; s++)
            if (tp_recv(&t, A * g, A * g + s, 1, T + (size_t)A * p * blk + (size_t)s * blk, blk) != (int64_t)blk) err = -2;
    if (st) st->rounds++;
    /* (2) Bruck among leaders on aggregates: T_A[0] = own aggregate; round k sends T_A[0..n_k)
     * to leader (A - 2^k) mod G, stored at T[2^k ..]; final aggregate j = T_A[(j - A) mod G] */
    for (int k = 0; k < K && !err; k++) {
        const int d = 1 << k, nk = (d < G - d) ? d : G - d;
        for (int A = 0; A < G && !err; A++)
            err = tp_send(&t, A * g, imod(A - d, G) * g, 2 + k, T + (size_t)A * p * blk, (size_t)nk * agg);
        for (int A = 0; A < G && !err; A++)
            if (tp_recv(&t, A * g, imod(A + d, G) * g, 2 + k, T + (size_t)A * p * blk + (size_t)d * agg,
                        (size_t)nk * agg) != (int64_t)((size_t)nk * agg)) err = -2;
        if (st) st->rounds++;
    }
    /* (3) leader unrotates into rank order and broadcasts to its node */
    for (int A = 0; A < G && !err; A++) {
        for (int j = 0; j < G; j++) memcpy(buf + (size_t)j * agg, T + (size_t)A * p * blk + (size_t)imod(j - A, G) * agg, agg);
        for (int s = 0; s < g && !err; s++) err = tp_send(&t, A * g, A * g + s, 64, buf, (size_t)p * blk);
    }
    for (int r = 0; r < p && !err; r++)
        if (tp_recv(&t, r, (r / g) * g, 64, recv + (size_t)r * p * blk, (size_t)p * blk) != (int64_t)((size_t)p * blk)) err = -2;
    if (st) st->rounds++;
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    free(T); free(buf);
    return err;
}

/* f2(iii) / north_star "Bruck ... pack/unpack for ... v-variants": Bruck alltoallv.  The
 * paper is silent; this follows C.4 item 2 with variable blocks: R1 T_r[i] =
 * the segment send_r sends to (r+i) mod p; round k packs the blocks with bit k of i set, in
 * increasing i, each preceded by an 8-byte length header (SPEC.md:258's in-band headers), to
 * (r+2^k) mod p, which unpacks them into the same indices; R3 recv_r[rd_r[j]] = T_r[(r-j)
 * mod p].  Messages per rank = ceil(log2 p), as for the uniform Bruck. */
int orc_alltoallv_bruck(int p, size_t w, const unsigned char *send, size_t sstride, const int64_t *sc,
                        const int64_t *sd, unsigned char *recv, size_t rstride, const int64_t *rc,
                        const int64_t *rd, orc_stats *st) {
    if (!v_args_ok(p, w, sstride, sc, sd, rstride, rc, rd)) return -1;
    unsigned char **T = (unsigned char **)calloc((size_t)p * p, sizeof(unsigned char *));
    size_t *Tn = (size_t *)calloc((size_t)p * p, sizeof(size_t));
    size_t cap = 8 * (size_t)p;
    for (int r = 0; r < p; r++)
        for (int j = 0; j < p; j++) cap += (size_t)sc[r * p + j] * w;
    unsigned char *pack = (unsigned char *)malloc(cap + 1);
    transport_t t;
    if (!T || !Tn || !pack || tp_init(&t, p, st)) { free(T); free(Tn); free(pack); return -1; }
    int err = 0;
    for (int r = 0; r < p; r++)                     /* R1 */
        for (int i = 0; i < p; i++) {
            int j = imod(r + i, p);
            size_t n = (size_t)sc[r * p + j] * w;
            T[r * p + i] = (unsigned char *)malloc(n + 1);
            Tn[r * p + i] = n;
            if (n) memcpy(T[r * p + i], send + (size_t)r * sstride + (size_t)sd[r * p + j] * w, n);
        }
    const int K = ceil_log2(p);
    for (int k = 0; k < K && !err; k++) {
        const int d = 1 << k;
        for (int r = 0; r < p && !err; r++) {      /* pack: [len][bytes] per block with bit k */
            size_t n = 0;
            for (int i = 0; i < p; i++)
                if ((i >> k) & 1) {
                    uint64_t len = Tn[r * p + i];
                    memcpy(pack + n, &len, 8);
                    if (len) memcpy(pack + n + 8, T[r * p + i], len);
                    n += 8 + len;
                }
            err = tp_send(&t, r, imod(r + d, p), k, pack, n);
        }
        for (int r = 0; r < p && !err; r++) {      /* unpack into the same indices */
            int64_t n = tp_recv(&t, r, imod(r - d, p), k, pack, cap);
            if (n < 0) { err = -2; break; }
            size_t o = 0;
            for (int i = 0; i < p && !err; i++)
                if ((i >> k) & 1) {
                    uint64_t len;
                    memcpy(&len, pack + o, 8);
                    free(T[r * p + i]);
                    T[r * p + i] = (unsigned char *)malloc(len + 1);
                    Tn[r * p + i] = len;
                    if (len) memcpy(T[r * p + i], pack + o + 8, len);
                    o += 8 + len;
                }
            if (o != (size_t)n) err = -2;
        }
        if (st) st->rounds++;
    }
    for (int r = 0; r < p && !err; r++)            /* R3 */
        for (int j = 0; j < p; j++) {
            const size_t n = Tn[r * p + imod(r - j, p)];
            if (n != (size_t)rc[r * p + j] * w) { err = -2; break; }
            if (n) memcpy(recv + (size_t)r * rstride + (size_t)rd[r * p + j] * w, T[r * p + imod(r - j, p)], n);
        }
    if (!err && tp_pending(&t)) err = -2;
    tp_free(&t);
    for (int i = 0; i < p * p; i++) free(T[i]);
    free(T); free(Tn); free(pack);
    return err;
}

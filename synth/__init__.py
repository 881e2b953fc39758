"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no exchange, rotation, scan or
schedule). It only produces payload bytes and count matrices from a seed, so
that the CPU oracle (``oracle/``) and the CUDA path
(``paper_2309_07337_b200``) can be fed identical inputs without sharing code.

Recipe (BASELINE.json configs[0..4]):

* ``mix64`` is the SplitMix64 finalizer.
* ``h32(seed, r, j, k)`` = low 32 bits of ``mix64(seed ^ mix64((r << 48) | (j << 32) | k))``
  with ``r, j < 2**16`` and ``k < 2**32``.
* cfg1 int32 word k of block (r -> j)      : ``h32(seed, r, j, k)``
* cfg2 uint8 byte t of rank r's contribution: byte ``t % 4`` (little endian) of
  ``h32(seed, r, 0, t // 4)``
* cfg3 float32 element k of block (r -> j) : ``((h32 >> 8) * 2**-23) - 1`` in [-1, 1), exact in fp32
* cfg4 int64 element k of segment (r -> j) : ``h32(.., 2k+1) << 32 | h32(.., 2k)``
* cfg5 bf16 element k of block (r -> j)    : Box-Muller in float64 from
  ``u1 = (h32(.., 2k) + 1) / 2**32`` and ``u2 = h32(.., 2k+1) / 2**32``, then
  round-to-nearest-even to bf16 (bit pattern returned as uint16).
* cfg4 counts: ``c[r][j] = h32(seed ^ 0xC0117, r, j, 0) % (2*mean_el + 1)``
  elements, then the ``floor(0.1 * p * p)`` pairs with the smallest
  ``h32(seed ^ 0x2E50, r, j, 0)`` are forced to 0 (ties by (r, j)).

All payloads are treated by the library as opaque bytes (BASELINE.json cfg3:
"treated as opaque bytes").
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK32 = np.uint64(0xFFFFFFFF)


def mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finalizer over a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def h32(seed: int, r, j, k) -> np.ndarray:
    """Vectorised h32(seed, r, j, k) as uint32 (broadcasts over r, j, k)."""
    r = np.asarray(r, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    k = np.asarray(k, dtype=np.uint64)
    x = (r << np.uint64(48)) | (j << np.uint64(32)) | k
    z = mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ mix64(x))
    return (z & _MASK32).astype(np.uint32)


def words(seed: int, r: int, j: int, n: int, k0: int = 0) -> np.ndarray:
    """n consecutive uint32 words h32(seed, r, j, k0..k0+n-1)."""
    return h32(seed, r, j, np.arange(k0, k0 + n, dtype=np.uint64))


def block_bytes(seed: int, r: int, j: int, nbytes: int) -> np.ndarray:
    """nbytes opaque bytes of block (r -> j): the little-endian bytes of words()."""
    n = (nbytes + 3) // 4
    return words(seed, r, j, n).view(np.uint8)[:nbytes].copy()


# ---- per-config payloads (BASELINE.json configs) -------------------------

def cfg1_block(seed: int, r: int, j: int, count: int = 8) -> np.ndarray:
    """cfg1: int32 words k=0..count-1 of block (r -> j); returned as uint32."""
    return words(seed, r, j, count)


def cfg2_contribution(seed: int, r: int, nbytes: int) -> np.ndarray:
    """cfg2: rank r's uint8 allgather contribution of nbytes bytes."""
    return block_bytes(seed, r, 0, nbytes)


def cfg3_block(seed: int, r: int, j: int, count: int) -> np.ndarray:
    """cfg3: float32 values in [-1, 1) of block (r -> j)."""
    h = words(seed, r, j, count)
    return ((h >> np.uint32(8)).astype(np.float64) * 2.0 ** -23 - 1.0).astype(np.float32)


def cfg4_segment(seed: int, r: int, j: int, count: int) -> np.ndarray:
    """cfg4: int64 elements of segment (r -> j)."""
    h = words(seed, r, j, 2 * count).astype(np.uint64)
    v = (h[1::2] << np.uint64(32)) | h[0::2]
    return v.view(np.int64)


def _f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float64 -> bf16 once, to nearest with ties to even (np.rint is RNE),
    on the bf16 grid of 8 significant bits; returns the bf16 bit patterns."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                       # x = m * 2**e, 0.5 <= |m| < 1
    q = np.ldexp(np.rint(m * 256.0), e - 8)  # exact in bf16 (and in float32)
    return (q.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def cfg5_block(seed: int, r: int, j: int, count: int) -> np.ndarray:
    """cfg5: bf16 N(0,1) values of block (r -> j) as uint16 bit patterns."""
    h = words(seed, r, j, 2 * count).astype(np.float64)
    u1 = (h[0::2] + 1.0) / 2.0 ** 32
    u2 = h[1::2] / 2.0 ** 32
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return _f64_to_bf16_bits(z)


def cfg4_counts(seed: int, p: int, mean_bytes: int, elem: int = 8) -> np.ndarray:
    """cfg4 count matrix c[r][j] in elements (int64), with floor(0.1 p^2) forced zeros."""
    mean_el = mean_bytes // elem
    r = np.arange(p, dtype=np.uint64)[:, None]
    j = np.arange(p, dtype=np.uint64)[None, :]
    c = (h32(seed ^ 0xC0117, r, j, 0).astype(np.int64) % (2 * mean_el + 1)).astype(np.int64)
    nz = int(0.1 * p * p)
    if nz:
        key = h32(seed ^ 0x2E50, r, j, 0).astype(np.int64)
        order = sorted(((int(key[a, b]), a, b) for a in range(p) for b in range(p)))
        for _, a, b in order[:nz]:
            c[a, b] = 0
    return c


# ---- generic process buffers ----------------------------------------------------------

def alltoall_sendbuf(seed: int, p: int, block: int, dtype: str = "bytes") -> np.ndarray:
    """(p, p*block) uint8 array: row r = rank r's sendbuf, block j -> rank j.

    dtype selects the config payload: 'bytes' (h32 words), 'f32' (cfg3),
    'bf16' (cfg5); block is in BYTES (must be a multiple of the element size).
    """
    out = np.empty((p, p * block), dtype=np.uint8)
    for r in range(p):
        for j in range(p):
            if dtype == "bytes":
                b = block_bytes(seed, r, j, block)
            elif dtype == "f32":
                b = cfg3_block(seed, r, j, block // 4).view(np.uint8)
            elif dtype == "bf16":
                b = cfg5_block(seed, r, j, block // 2).view(np.uint8)
            elif dtype == "i64":
                b = cfg4_segment(seed, r, j, block // 8).view(np.uint8)
            else:
                raise ValueError(dtype)
            out[r, j * block:(j + 1) * block] = b
    return out


def allgather_sendbuf(seed: int, p: int, nbytes: int) -> np.ndarray:
    """(p, nbytes) uint8: row r = rank r's contribution (cfg2 payload)."""
    out = np.empty((p, nbytes), dtype=np.uint8)
    for r in range(p):
        out[r] = cfg2_contribution(seed, r, nbytes)
    return out


def alltoallv_buffers(seed: int, counts: np.ndarray, elem: int = 8, packed: bool = True):
    """Send buffers and displacement arrays for an alltoallv with count matrix counts[r][j].

    Returns (send (p, S) uint8, sendcounts, sdispls, recvcounts, rdispls, S, Rcap) where
    counts/displs are (p, p) int64 in ELEMENTS.  packed=True: exclusive prefix sums
    (SURVEY.md Q10); packed=False: segments placed with seeded gaps (any non-overlapping
    displacement is legal MPI).
    """
    p = counts.shape[0]
    sc = counts.astype(np.int64)
    rc = counts.T.copy().astype(np.int64)
    if packed:
        sd = np.zeros_like(sc)
        rd = np.zeros_like(rc)
        sd[:, 1:] = np.cumsum(sc, axis=1)[:, :-1]
        rd[:, 1:] = np.cumsum(rc, axis=1)[:, :-1]
    else:
        gap_s = (h32(seed ^ 0x6A9, np.arange(p)[:, None], np.arange(p)[None, :], 0) % 3).astype(np.int64)
        gap_r = (h32(seed ^ 0x6AA, np.arange(p)[:, None], np.arange(p)[None, :], 0) % 3).astype(np.int64)
        # reverse placement order to exercise non-monotone displacements
        sd = np.zeros_like(sc)
        rd = np.zeros_like(rc)
        for r in range(p):
            off = 0
            for j in reversed(range(p)):
                off += gap_s[r, j]
                sd[r, j] = off
                off += sc[r, j]
            off = 0
            for j in reversed(range(p)):
                off += gap_r[r, j]
                rd[r, j] = off
                off += rc[r, j]
    S = int(max(1, (sd + sc).max())) * elem
    Rcap = int(max(1, (rd + rc).max())) * elem
    send = np.zeros((p, S), dtype=np.uint8)
    for r in range(p):
        for j in range(p):
            n = int(sc[r, j])
            if n:
                seg = cfg4_segment(seed, r, j, (n * elem + 7) // 8).view(np.uint8)[: n * elem]
                o = int(sd[r, j]) * elem
                send[r, o:o + n * elem] = seg
    return send, sc, sd, rc, rd, S, Rcap


# ---- f1: neighborhood topologies -------------------------------------
# Graph dicts as in oracle.neighbor_*: global, rank-major edge lists with packed
# displacements (exclusive prefix sums in edge order).  Element payloads are a pure
# function of the element's global index (h32 of the index), so equal indices carry equal
# values everywhere -- the precondition of the locality-aware variant.

def _pack(counts_per_rank):
    """Exclusive prefix sums of each rank's edge counts (packed displacements)."""
    out = []
    for cs in counts_per_rank:
        d, acc = [], 0
        for c in cs:
            d.append(acc)
            acc += c
        out.append(d)
    return out


def graph_from_edges(p, edges):
    """edges: list of (src, dst, ids) with ids a list of global indices (count = len).
    Out-edges of a rank are in list order; in-edges of a rank are in list order too.
    Returns (graph, send_idx, recv_idx)."""
    outs = [[] for _ in range(p)]
    ins = [[] for _ in range(p)]
    for s, d, ids in edges:
        outs[s].append((d, list(ids)))
        ins[d].append((s, list(ids)))
    sd = _pack([[len(i) for _, i in o] for o in outs])
    rd = _pack([[len(i) for _, i in o] for o in ins])
    g = {"indeg": np.array([len(i) for i in ins], np.int32),
         "src": np.array([s for i in ins for s, _ in i], np.int32),
         "rc": np.array([len(ids) for i in ins for _, ids in i], np.int64),
         "rd": np.array([x for r in rd for x in r], np.int64),
         "outdeg": np.array([len(o) for o in outs], np.int32),
         "dst": np.array([d for o in outs for d, _ in o], np.int32),
         "sc": np.array([len(ids) for o in outs for _, ids in o], np.int64),
         "sd": np.array([x for r in sd for x in r], np.int64)}
    send_idx = np.array([x for o in outs for _, ids in o for x in ids], np.int64)
    recv_idx = np.array([x for i in ins for _, ids in i for x in ids], np.int64)
    return g, send_idx, recv_idx


def neighbor_buffers(seed, p, gr, send_idx, w=8, canary=0xA5):
    """Send rows (packed per out-edge; element value = h32-based function of its global
    index, w bytes) and a canary-filled recv buffer sized for the in-edges."""
    sc, sd, rc, rd = gr["sc"], gr["sd"], gr["rc"], gr["rd"]
    ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])])
    S = max(1, max((int((sd[ooff[r]:ooff[r + 1]] + sc[ooff[r]:ooff[r + 1]]).max()) if ooff[r + 1] > ooff[r] else 0)
                   for r in range(p))) * w
    R = max(1, max((int((rd[ioff[r]:ioff[r + 1]] + rc[ioff[r]:ioff[r + 1]]).max()) if ioff[r + 1] > ioff[r] else 0)
                   for r in range(p))) * w
    send = np.zeros((p, S), np.uint8)
    e0 = 0
    for r in range(p):
        for e in range(ooff[r], ooff[r + 1]):
            n = int(sc[e])
            ids = send_idx[e0:e0 + n].astype(np.uint64)
            e0 += n
            if n:
                words = (w + 3) // 4
                vals = np.stack([h32(seed, 0, 0, ids * np.uint64(words) + np.uint64(k)) for k in range(words)], 1)
                send[r, int(sd[e]) * w:(int(sd[e]) + n) * w] = vals.astype(np.uint32).view(np.uint8).reshape(n, -1)[:, :w].reshape(-1)
    return send, np.full((p, R), canary, np.uint8)


def ring_edges(p, count):
    """SPEC.md:300-303 ring: rank r sends `count` elements to r-1 and r+1 (ids unique per edge)."""
    edges = []
    for r in range(p):
        for d in ((r - 1) % p, (r + 1) % p):
            edges.append((r, d, [(r * p + d) * count + k for k in range(count)]))
    return edges


def stencil_edges(px, py, nx, ny, corners=True):
    """2-D halo exchange: an nx x ny grid of points (global index y*nx + x) split into
    px x py rank blocks (rank = by*px + bx).  Each rank sends the boundary points a
    neighbouring block needs: one row/column to each edge neighbour (5-point) and, with
    corners, its corner point to each diagonal neighbour (9-point).  A corner point thus goes
    to three ranks -- duplicate indices across a node boundary when those ranks share a node."""
    bw, bh = nx // px, ny // py
    edges = []
    for by in range(py):
        for bx in range(px):
            r = by * px + bx
            x0, y0 = bx * bw, by * bh
            x1, y1 = x0 + bw - 1, y0 + bh - 1
            nbrs = []
            if bx > 0: nbrs.append(((by, bx - 1), [y * nx + x0 for y in range(y0, y1 + 1)]))
            if bx < px - 1: nbrs.append(((by, bx + 1), [y * nx + x1 for y in range(y0, y1 + 1)]))
            if by > 0: nbrs.append(((by - 1, bx), [y0 * nx + x for x in range(x0, x1 + 1)]))
            if by < py - 1: nbrs.append(((by + 1, bx), [y1 * nx + x for x in range(x0, x1 + 1)]))
            if corners:
                for dy, dx, cx, cy in ((-1, -1, x0, y0), (-1, 1, x1, y0), (1, -1, x0, y1), (1, 1, x1, y1)):
                    if 0 <= by + dy < py and 0 <= bx + dx < px:
                        nbrs.append(((by + dy, bx + dx), [cy * nx + cx]))
            for (ny_, nx_), ids in nbrs:
                edges.append((r, ny_ * px + nx_, ids))
    return edges


def random_edges(seed, p, max_deg, max_count, idx_space):
    """Random multigraph: each rank gets up to max_deg out-edges (repeats and self-edges
    allowed), counts 0..max_count, element ids drawn from [0, idx_space) (duplicates
    across and within edges)."""
    rng = np.random.default_rng(seed)
    edges = []
    for r in range(p):
        for _ in range(int(rng.integers(0, max_deg + 1))):
            d = int(rng.integers(0, p))
            n = int(rng.integers(0, max_count + 1))
            edges.append((r, d, [int(x) for x in rng.integers(0, idx_space, n)]))
    return edges


def spmv_edges(seed, p, m, k, deg, contiguous=False):
    """Sparse-matrix halo (the neighbourhood collectives' use case): rank r owns m boundary
    values (global ids r*m .. r*m+m-1); every rank q needs k of them from each of `deg`
    distinct other ranks -- a random subset (sorted, without replacement), or with
    contiguous=True a random window of k consecutive ids (banded / reordered matrices).
    Ranks of one group needing the same value create the duplicates the locality-aware
    variant removes."""
    rng = np.random.default_rng(seed)
    need = {}
    for q in range(p):
        owners = rng.choice([r for r in range(p) if r != q], size=min(deg, p - 1), replace=False)
        for r in owners:
            if contiguous:
                s0 = int(rng.integers(0, m - min(k, m) + 1))
                need[(int(r), q)] = list(range(int(r) * m + s0, int(r) * m + s0 + min(k, m)))
            else:
                need[(int(r), q)] = sorted(int(r) * m + int(x) for x in rng.choice(m, size=min(k, m), replace=False))
    return [(r, q, need[(r, q)]) for (r, q) in sorted(need)]

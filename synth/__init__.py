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

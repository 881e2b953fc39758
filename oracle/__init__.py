"""mpxa CPU oracle (ctypes wrapper over oracle/mpxa_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg
and ``--impl reference`` arm) may import this package.  The product package
``paper_2309_07337_b200`` never imports it and shares no code with it.

Every function takes/returns numpy arrays laid out one row per rank (see the C file's
header for the exact layouts and the paper passages each function follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpxa_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no vectorisation flags needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "ppn", "msgs", "bytes", "intra_msgs", "inter_msgs", "intra_bytes", "inter_bytes",
        "max_msgs_per_rank", "rounds")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I, Z = ctypes.c_int, ctypes.c_size_t
        S = ctypes.POINTER(Stats)
        sig = {
            "orc_alltoall_definition": [I, Z, P, P],
            "orc_allgather_definition": [I, Z, P, P],
            "orc_allgather_definition_rows": [I, Z, P, P, I, I],
            "orc_alltoallv_definition": [I, Z, P, Z, P, P, P, Z, P, P],
            "orc_alltoallv_pairwise": [I, Z, P, Z, P, P, P, Z, P, P, S],
            "orc_alltoall_pairwise": [I, Z, P, P, S],
            "orc_alltoall_bruck": [I, Z, P, P, I, P, S],
            "orc_allgather_bruck": [I, Z, P, P, I, P, S],
            "orc_allgather_ring": [I, Z, P, P, S],
            "orc_allgather_direct": [I, Z, P, P, S],
            "orc_alltoallv_hier": [I, I, Z, P, Z, P, P, P, Z, P, P, S],
            "orc_alltoall_hier": [I, I, Z, P, P, S],
            "orc_counts_exchange": [I, P, P, P, S],
            "orc_neighbor_definition": [I, Z, P, P, P, P, P, Z, P, P, P, P, P, Z],
            "orc_neighbor_standard": [I, Z, P, P, P, P, P, Z, P, P, P, P, P, Z, S],
            "orc_neighbor_locality": [I, I, Z, P, P, P, P, P, P, Z, P, P, P, P, P, P, Z, S, P],
            "orc_part_arrived": [I, Z, I, Z, P, P],
            "orc_allgather_hier": [I, I, Z, P, P, S],
            "orc_alltoallv_bruck": [I, Z, P, Z, P, P, P, Z, P, P, S],
            "orc_part_cycle": [I, Z, I, Z, P, P, P, P, S],
        }
        for name, args in sig.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _u8(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _check(rc, name):
    if rc != 0:
        raise RuntimeError(f"oracle {name} failed with {rc}")


# ---- definitions ----------------------------------------------------

def alltoall_definition(send: np.ndarray) -> np.ndarray:
    """send: (p, p*blk) uint8 -> recv (p, p*blk) with recv_r[j] = send_j[r]."""
    send = _u8(send)
    p = send.shape[0]
    blk = send.shape[1] // p if p else 0
    recv = np.zeros_like(send)
    _check(lib().orc_alltoall_definition(p, blk, _ptr(send), _ptr(recv)), "alltoall_definition")
    return recv


def allgather_definition(send: np.ndarray) -> np.ndarray:
    """send: (p, blk) uint8 -> recv (p, p*blk) with recv_r[j] = send_j."""
    send = _u8(send)
    p, blk = send.shape
    recv = np.zeros((p, p * blk), dtype=np.uint8)
    _check(lib().orc_allgather_definition(p, blk, _ptr(send), _ptr(recv)), "allgather_definition")
    return recv


def allgather_definition_threaded(send: np.ndarray, nthreads: int, recv: np.ndarray = None) -> np.ndarray:
    """allgather_definition with the receiving ranks split over `nthreads` host threads, each
    calling orc_allgather_definition_rows on its own rows (ctypes releases the GIL during
    the call, so the threads run concurrently).  Timing aid for the host baseline."""
    from concurrent.futures import ThreadPoolExecutor
    send = _u8(send)
    p, blk = send.shape
    if recv is None:
        recv = np.zeros((p, p * blk), dtype=np.uint8)
    T = max(1, min(int(nthreads), p))
    bounds = [(p * t // T, p * (t + 1) // T) for t in range(T)]
    L = lib()
    with ThreadPoolExecutor(T) as ex:
        rcs = list(ex.map(lambda b: L.orc_allgather_definition_rows(p, blk, _ptr(send), _ptr(recv), b[0], b[1]),
                          bounds))
    for rc in rcs:
        _check(rc, "allgather_definition_rows")
    return recv


def _v_arrays(sc, sd, rc, rd):
    return [np.ascontiguousarray(x, dtype=np.int64) for x in (sc, sd, rc, rd)]


def alltoallv_definition(send, sc, sd, rc, rd, w, recv_init):
    """Returns a copy of recv_init (p, rstride) with the received ranges written."""
    send = _u8(send)
    sc, sd, rc, rd = _v_arrays(sc, sd, rc, rd)
    recv = np.array(_u8(recv_init), copy=True)
    p = send.shape[0]
    _check(lib().orc_alltoallv_definition(p, w, _ptr(send), send.shape[1], _ptr(sc), _ptr(sd),
                                          _ptr(recv), recv.shape[1], _ptr(rc), _ptr(rd)),
           "alltoallv_definition")
    return recv


# ---- variant simulations --------------------------------------------

def alltoall(send: np.ndarray, variant: str = "pairwise", g: int = 0, stop_stage: int = -1,
             ppn: int = 0):
    """Simulate one alltoall variant.  Returns (recv, T or None, stats dict)."""
    send = _u8(send)
    p = send.shape[0]
    blk = send.shape[1] // p if p else 0
    recv = np.zeros_like(send)
    st = Stats(ppn=ppn)
    T = None
    L = lib()
    if variant == "pairwise":
        rc = L.orc_alltoall_pairwise(p, blk, _ptr(send), _ptr(recv), ctypes.byref(st))
    elif variant == "bruck":
        T = np.zeros_like(send)
        rc = L.orc_alltoall_bruck(p, blk, _ptr(send), _ptr(recv), stop_stage, _ptr(T), ctypes.byref(st))
    elif variant == "hier":
        st.ppn = g
        rc = L.orc_alltoall_hier(p, g, blk, _ptr(send), _ptr(recv), ctypes.byref(st))
    else:
        raise ValueError(variant)
    _check(rc, "alltoall/" + variant)
    return recv, T, st.as_dict()


def allgather(send: np.ndarray, variant: str = "bruck", stop_stage: int = -1, ppn: int = 0, g: int = 0):
    """send (p, blk) -> (recv (p, p*blk), T or None, stats)."""
    send = _u8(send)
    p, blk = send.shape
    recv = np.zeros((p, p * blk), dtype=np.uint8)
    st = Stats(ppn=ppn)
    T = None
    L = lib()
    if variant == "bruck":
        T = np.zeros((p, p * blk), dtype=np.uint8)
        rc = L.orc_allgather_bruck(p, blk, _ptr(send), _ptr(recv), stop_stage, _ptr(T), ctypes.byref(st))
    elif variant == "ring":
        rc = L.orc_allgather_ring(p, blk, _ptr(send), _ptr(recv), ctypes.byref(st))
    elif variant in ("direct", "pairwise"):
        rc = L.orc_allgather_direct(p, blk, _ptr(send), _ptr(recv), ctypes.byref(st))
    elif variant == "hier":
        st.ppn = g
        rc = L.orc_allgather_hier(p, g, blk, _ptr(send), _ptr(recv), ctypes.byref(st))
    else:
        raise ValueError(variant)
    _check(rc, "allgather/" + variant)
    return recv, T, st.as_dict()


def alltoallv(send, sc, sd, rc, rd, w, recv_init, variant: str = "pairwise", g: int = 0,
              ppn: int = 0):
    send = _u8(send)
    sc, sd, rc_, rd = _v_arrays(sc, sd, rc, rd)
    recv = np.array(_u8(recv_init), copy=True)
    p = send.shape[0]
    st = Stats(ppn=ppn)
    L = lib()
    args = (_ptr(send), send.shape[1], _ptr(sc), _ptr(sd), _ptr(recv), recv.shape[1], _ptr(rc_), _ptr(rd))
    if variant == "pairwise":
        r = L.orc_alltoallv_pairwise(p, w, *args, ctypes.byref(st))
    elif variant == "hier":
        st.ppn = g
        r = L.orc_alltoallv_hier(p, g, w, *args, ctypes.byref(st))
    elif variant == "bruck":
        r = L.orc_alltoallv_bruck(p, w, *args, ctypes.byref(st))
    else:
        raise ValueError(variant)
    _check(r, "alltoallv/" + variant)
    return recv, st.as_dict()


def counts_exchange(sendcounts: np.ndarray):
    """sendcounts (p, p) int64 -> (recvcounts, rdispls, stats)."""
    sc = np.ascontiguousarray(sendcounts, dtype=np.int64)
    p = sc.shape[0]
    rc = np.zeros_like(sc)
    rd = np.zeros_like(sc)
    st = Stats()
    _check(lib().orc_counts_exchange(p, _ptr(sc), _ptr(rc), _ptr(rd), ctypes.byref(st)), "counts_exchange")
    return rc, rd, st.as_dict()


# ---- f1: neighborhood alltoallv --------------------
# A graph is a dict of numpy arrays (global view, rank-major edge lists):
#   indeg (p,) int32, src/rc/rd (sum indeg,) int32/int64/int64 -- in-edges in order
#   outdeg (p,) int32, dst/sc/sd (sum outdeg,) int32/int64/int64 -- out-edges in order
# Locality variant: send_idx / recv_idx, one int64 global index per element, edge by edge.

def _graph_args(gr):
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
    return (i32(gr["indeg"]), i32(gr["src"]), i64(gr["rc"]), i64(gr["rd"]),
            i32(gr["outdeg"]), i32(gr["dst"]), i64(gr["sc"]), i64(gr["sd"]))


def neighbor_definition(send, recv_init, w, gr):
    """MPI_Neighbor_alltoallv result: recv_init copy with every in-edge's range written."""
    send = _u8(send)
    recv = np.array(_u8(recv_init), copy=True)
    indeg, src, rc, rd, outdeg, dst, sc, sd = a = _graph_args(gr)
    p = send.shape[0]
    _check(lib().orc_neighbor_definition(p, w, _ptr(indeg), _ptr(src), _ptr(rc), _ptr(rd), _ptr(recv),
                                         recv.shape[1], _ptr(outdeg), _ptr(dst), _ptr(sc), _ptr(sd),
                                         _ptr(send), send.shape[1]), "neighbor_definition")
    del a
    return recv


def neighbor(send, recv_init, w, gr, variant="standard", g=0, send_idx=None, recv_idx=None, ppn=0):
    """Simulate the standard or the locality-aware (variant='locality', groups of g ranks)
    persistent neighbor alltoallv.  Returns (recv, stats dict); stats gains 'inter_values'
    (index/value records crossing group boundaries) for the locality variant."""
    send = _u8(send)
    recv = np.array(_u8(recv_init), copy=True)
    indeg, src, rc, rd, outdeg, dst, sc, sd = _graph_args(gr)
    p = send.shape[0]
    st = Stats(ppn=ppn or g or p)
    L = lib()
    if variant == "standard":
        r = L.orc_neighbor_standard(p, w, _ptr(indeg), _ptr(src), _ptr(rc), _ptr(rd), _ptr(recv), recv.shape[1],
                                    _ptr(outdeg), _ptr(dst), _ptr(sc), _ptr(sd), _ptr(send), send.shape[1],
                                    ctypes.byref(st))
        _check(r, "neighbor/standard")
        return recv, st.as_dict()
    if variant != "locality":
        raise ValueError(variant)
    si = np.ascontiguousarray(send_idx, dtype=np.int64)
    ri = np.ascontiguousarray(recv_idx, dtype=np.int64)
    iv = ctypes.c_int64(0)
    r = L.orc_neighbor_locality(p, g, w, _ptr(indeg), _ptr(src), _ptr(rc), _ptr(rd), _ptr(ri), _ptr(recv),
                                recv.shape[1], _ptr(outdeg), _ptr(dst), _ptr(sc), _ptr(sd), _ptr(si), _ptr(send),
                                send.shape[1], ctypes.byref(st), ctypes.byref(iv))
    if r == -3:
        raise ValueError("inconsistent recv_indices (locality handshake)")
    _check(r, "neighbor/locality")
    d = st.as_dict()
    d["inter_values"] = int(iv.value)
    return recv, d


# ---- f3: partitioned point-to-point ----------------

def part_arrived(n_s, bs, n_r, br, delivered):
    """Parrived of every receiver partition, given which sender partitions were delivered."""
    d = np.ascontiguousarray(np.asarray(delivered, dtype=np.uint8))
    out = np.zeros(n_r, np.uint8)
    _check(lib().orc_part_arrived(n_s, bs, n_r, br, _ptr(d), _ptr(out)), "part_arrived")
    return out.astype(bool)


def part_cycle(send, n_s, n_r, order):
    """One partitioned cycle with Pready in `order`: returns (recv bytes, trace (n_s, n_r) of
    Parrived after each delivery, stats)."""
    send = np.ascontiguousarray(send, dtype=np.uint8)
    total = send.size
    bs, br = total // n_s, total // n_r
    recv = np.zeros_like(send)
    order = np.ascontiguousarray(order, dtype=np.int32)
    trace = np.zeros((n_s, n_r), np.uint8)
    st = Stats()
    _check(lib().orc_part_cycle(n_s, bs, n_r, br, _ptr(send), _ptr(recv), _ptr(order), _ptr(trace),
                                ctypes.byref(st)), "part_cycle")
    return recv, trace.astype(bool), st.as_dict()

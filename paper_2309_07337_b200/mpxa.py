"""Thin Python binding over libmpxa.so (include/mpxa.h, include/mpxa_plan.h).

Argument marshalling only: every step of every collective runs in the library's sm_100a
kernels.  PyTorch supplies device memory (tensors), streams and -- for multi-process
communicators -- the process group used by the bootstrap all-gather.  There is no CPU or
PyTorch fallback: if libmpxa.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import weakref
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPXA_LIB") or os.path.join(_HERE, "libmpxa.so")   # MPXA_LIB: tuning builds

# ---- constants (mirror include/mpxa.h) ------------------------------------------------
SUCCESS, ERR_ARG, ERR_ALGO, ERR_LIFECYCLE, ERR_TOPOLOGY, ERR_MISMATCH, ERR_CUDA, ERR_TIMEOUT, \
    ERR_NOMEM, ERR_UNREGISTERED = range(10)
OP_ALLTOALL, OP_ALLTOALLV, OP_ALLGATHER, OP_NEIGHBOR_ALLTOALLV = 0, 1, 2, 3
ALGO = {"default": 0, "pairwise": 1, "bruck": 2, "hier": 3, "ring": 4, "locality": 5}
ALGO_NAME = {v: k for k, v in ALGO.items()}
OPS = {"alltoall": OP_ALLTOALL, "alltoallv": OP_ALLTOALLV, "allgather": OP_ALLGATHER,
       "neighbor_alltoallv": OP_NEIGHBOR_ALLTOALLV}


class MpxaError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = _lib().mpxa_error_string(status).decode() if _LIB is not None else str(status)
        super().__init__(f"{what}: mpxa status {status} ({msg})")


BOOT_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


class InitArgs(ctypes.Structure):
    _fields_ = [("nprocs", ctypes.c_int), ("proc", ctypes.c_int), ("ranks_per_proc", ctypes.c_int),
                ("device", ctypes.c_int), ("group_size", ctypes.c_int), ("emulate_gpus", ctypes.c_int),
                ("bootstrap_allgather", BOOT_FN), ("ctx", ctypes.c_void_p),
                ("heap_bytes", ctypes.c_size_t), ("timeout_s", ctypes.c_double)]


class PlanMove(ctypes.Structure):
    _fields_ = [("src_off", ctypes.c_int64), ("dst_off", ctypes.c_int64), ("len", ctypes.c_int64),
                ("flow", ctypes.c_uint32), ("src_rank", ctypes.c_uint16), ("dst_rank", ctypes.c_uint16),
                ("src_kind", ctypes.c_uint8), ("dst_kind", ctypes.c_uint8),
                ("fanout", ctypes.c_uint8), ("pad", ctypes.c_uint8 * 5)]


class PlanStep(ctypes.Structure):
    _fields_ = [("move_begin", ctypes.c_int32), ("move_end", ctypes.c_int32),
                ("signal_mask", ctypes.c_uint32), ("wait_mask", ctypes.c_uint32),
                ("total_len", ctypes.c_int64), ("max_len", ctypes.c_int64), ("flow_index", ctypes.c_int32),
                ("dense_base", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("nsteps", "work_units", "max_move", "max_step_units", "signals", "total_moves", "nflows",
                 "max_step_moves")]


# every symbol of include/mpxa.h and include/mpxa_plan.h, with its ctypes signature
_P, _I, _Z, _U64P = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint64)
SIGNATURES = {
    "mpxa_init": ([_P, ctypes.POINTER(InitArgs)], _I),
    "mpxa_finalize": ([_P], _I),
    "mpxa_comm_size": ([_P, ctypes.POINTER(_I)], _I),
    "mpxa_comm_rank0": ([_P, ctypes.POINTER(_I)], _I),
    "mpxa_comm_check": ([_P], _I),
    "mpxa_launch_count": ([_P, _U64P], _I),
    "mpxa_register": ([_P, _P, _Z], _I),
    "mpxa_deregister": ([_P, _P], _I),
    "mpxa_alltoall": ([_P, _Z, _Z, _P, _P, _P], _I),
    "mpxa_allgather": ([_P, _Z, _Z, _P, _P, _P], _I),
    "mpxa_alltoallv": ([_P, _P, _P, _Z, _P, _P, _P, _Z, _Z, _P, _P], _I),
    "mpxa_alltoall_algo": ([_P, _Z, _Z, _P, _I, _P, _P], _I),
    "mpxa_allgather_algo": ([_P, _Z, _Z, _P, _I, _P, _P], _I),
    "mpxa_alltoallv_algo": ([_P, _P, _P, _Z, _P, _P, _P, _Z, _Z, _I, _P, _P], _I),
    "mpxa_alltoallv_counts": ([_P, _P, _P, _P, _P], _I),
    "mpxa_alltoall_bruck_stage": ([_P, _Z, _Z, _P, _I, _P, _P], _I),
    "mpxa_allgather_bruck_stage": ([_P, _Z, _Z, _P, _I, _P, _P], _I),
    "mpxa_alltoall_init": ([_P, _Z, _Z, _P, _I, _P, _P, _P], _I),
    "mpxa_allgather_init": ([_P, _Z, _Z, _P, _I, _P, _P, _P], _I),
    "mpxa_alltoallv_init": ([_P, _P, _P, _Z, _P, _P, _P, _Z, _Z, _I, _P, _P, _P], _I),
    "mpxa_start": ([_P, _P], _I),
    "mpxa_wait": ([_P, _P], _I),
    "mpxa_request_free": ([_P], _I),
    "mpxa_request_algorithm": ([_P, ctypes.POINTER(_I)], _I),
    "mpxa_set_algorithm": ([_P, _I, _I], _I),
    "mpxa_get_algorithm": ([_P, _I, _Z, ctypes.POINTER(_I)], _I),
    "mpxa_list_algorithms": ([_I, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "mpxa_load_selector": ([_P, ctypes.c_char_p], _I),
    "mpxa_config_digest": ([_P, _U64P], _I),
    "mpxa_error_string": ([_I], ctypes.c_char_p),
    "mpxa_algo_name": ([_I], ctypes.c_char_p),
    "mpxa_plan_build": ([_I, _I, _I, _I, _I, _I, _I, _P, _P, _P, ctypes.POINTER(_P)], _I),
    "mpxa_dist_graph_create_adjacent": ([_P, _P, _P, _P, _P, _P, _P, _P, _I, ctypes.POINTER(_P)], _I),
    "mpxa_topo_free": ([ctypes.POINTER(_P)], _I),
    "mpxa_neighbor_alltoallv_init": ([_P, _P, _P, _Z, _P, _P, _P, _Z, _Z, _P, _P, ctypes.POINTER(_P)], _I),
    "mpxa_neighbor_alltoallv_locality_init": ([_P, _P, _P, _Z, _P, _P, _P, _Z, _Z, _P, _P, _P, _P,
                                               ctypes.POINTER(_P)], _I),
    "mpxa_neighbor_alltoallv": ([_P, _P, _P, _Z, _P, _P, _P, _Z, _Z, _P, _P], _I),
    "mpxa_psend_init": ([_P, _I, _Z, _Z, _I, _I, _I, _P, _P, ctypes.POINTER(_P)], _I),
    "mpxa_precv_init": ([_P, _I, _Z, _Z, _I, _I, _I, _P, _P, ctypes.POINTER(_P)], _I),
    "mpxa_pmatch": ([_P], _I),
    "mpxa_pready": ([_P, _I, _P], _I),
    "mpxa_pready_range": ([_P, _I, _I, _P], _I),
    "mpxa_parrived": ([_P, _I, ctypes.POINTER(_I)], _I),
    "mpxa_parrived_wait": ([_P, _I, _I, _P], _I),
    "mpxa_psend_device": ([_P, _P, _Z], _I),
    "mpxa_plan_build_neighbor": ([_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_P)], _I),
    "mpxa_plan_eager": ([_P, _Z, ctypes.POINTER(_P)], _I),
    "mpxa_plan_info": ([_P, ctypes.POINTER(PlanInfo)], _I),
    "mpxa_plan_steps": ([_P, _I, _P, ctypes.POINTER(_I)], _I),
    "mpxa_plan_moves": ([_P, _I, _P, ctypes.POINTER(_I)], _I),
    "mpxa_plan_free": ([_P], _I),
}

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libmpxa.so not built at {LIB_PATH}: run `python __graft_entry__.py` "
                              "(build()) -- there is no fallback implementation")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            if os.environ.get("MPXA_LIB") and not hasattr(lib, name):
                continue   # an older tuning build (MPXA_LIB) may predate a symbol
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _LIB = lib
    return _LIB


def lib():
    return _lib()


def _ck(status: int, what: str):
    if status != SUCCESS:
        raise MpxaError(status, what)


def _algo(a) -> int:
    if a is None:
        return 0
    return ALGO[a] if isinstance(a, str) else int(a)


def _stream(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


_PTRS = {}   # id(ndarray) -> (weakref, address): repeated calls with the same arrays


def _host_i64(a):
    if type(a) is np.ndarray and a.dtype == np.int64 and a.flags.c_contiguous:   # fast path
        e = _PTRS.get(id(a))
        if e is not None and e[0]() is a:
            return a, e[1]
        addr = a.__array_interface__["data"][0]
        if len(_PTRS) > 256:
            _PTRS.clear()
        _PTRS[id(a)] = (weakref.ref(a), addr)
        return a, addr
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    return a, a.ctypes.data_as(ctypes.c_void_p)


def _i64_arg(a):
    """(keep-alive, pointer) of an int64 array argument: a CUDA int64 tensor is passed as a
    device pointer (the library copies it), anything else as a host array."""
    if hasattr(a, "is_cuda") and a.is_cuda:
        import torch
        if a.dtype != torch.int64 or not a.is_contiguous():
            raise ValueError("device counts / displacements must be contiguous int64 tensors")
        return a, ctypes.c_void_p(a.data_ptr())
    return _host_i64(a)


def list_algorithms(op: str):
    n = ctypes.c_int(8)
    out = (ctypes.c_int * 8)()
    _ck(_lib().mpxa_list_algorithms(OPS[op], out, ctypes.byref(n)), "list_algorithms")
    return [ALGO_NAME[out[i]] for i in range(n.value)]


class Request:
    """Persistent collective (MPIX_Request analog): start()/wait() any number of times."""

    def __init__(self, comm: "Comm", handle: int, keep):
        self.comm = comm
        self.handle = ctypes.c_void_p(handle)
        self._keep = keep   # keep bound tensors / host arrays alive

    def start(self, stream=None):
        _ck(_lib().mpxa_start(self.handle, _stream(stream)), "start")

    def wait(self, stream=None):
        _ck(_lib().mpxa_wait(self.handle, _stream(stream)), "wait")

    @property
    def algorithm(self) -> str:
        a = ctypes.c_int()
        _ck(_lib().mpxa_request_algorithm(self.handle, ctypes.byref(a)), "request_algorithm")
        return ALGO_NAME[a.value]

    def free(self):
        if self.handle:
            h = ctypes.c_void_p(self.handle.value)
            _ck(_lib().mpxa_request_free(ctypes.byref(h)), "request_free")
            self.handle = None


class Comm:
    """MPIX_Comm analog.

    Single process (pg None or world size 1): all p = ranks_per_proc ranks live on this
    device; buffers are rank-major [R][per-rank].  emulate_gpus = G > 1 splits them over G
    virtual GPUs that run the multi-GPU protocol (flags, CTS, peer-style stores) in one
    cooperative launch.  Multi-process (pg with world size > 1): one process per GPU,
    bootstrap all-gather over a gloo group.
    """

    def __init__(self, ranks_per_proc: int = 1, device: Optional[int] = None, group_size: int = 0,
                 emulate_gpus: int = 0, pg=None, heap_bytes: int = 0, timeout_s: float = 0.0):
        import torch
        self.handle = ctypes.c_void_p()
        nprocs, proc = 1, 0
        self._boot = None
        if pg is not None:
            import torch.distributed as dist
            nprocs, proc = dist.get_world_size(pg), dist.get_rank(pg)
            if nprocs > 1:
                gloo = pg if dist.get_backend(pg) == "gloo" else dist.new_group(backend="gloo")
                self._boot = make_bootstrap(gloo, nprocs)
        if device is None:
            device = torch.cuda.current_device()
        args = InitArgs(nprocs=nprocs, proc=proc, ranks_per_proc=ranks_per_proc, device=device,
                        group_size=group_size, emulate_gpus=emulate_gpus,
                        bootstrap_allgather=self._boot if self._boot else BOOT_FN(),
                        ctx=None, heap_bytes=heap_bytes, timeout_s=timeout_s)
        _ck(_lib().mpxa_init(ctypes.byref(self.handle), ctypes.byref(args)), "init")
        self.R = ranks_per_proc
        # group size g of the hierarchical variants (default: the ranks of one (virtual) GPU)
        self.g = group_size if group_size > 0 else (ranks_per_proc // emulate_gpus if emulate_gpus > 1
                                                    else ranks_per_proc)
        self.nprocs = nprocs
        self.proc = proc
        p = ctypes.c_int()
        _ck(_lib().mpxa_comm_size(self.handle, ctypes.byref(p)), "comm_size")
        self.p = p.value
        self.device = device

    # ---- introspection -------------------------------------------------------------
    def launch_count(self) -> int:
        n = ctypes.c_uint64()
        _ck(_lib().mpxa_launch_count(self.handle, ctypes.byref(n)), "launch_count")
        return n.value

    # bits of mpxa__last_launch (test hook, not part of the C ABI headers)
    PATH_BITS = {"small": 1, "eager": 2, "var": 4, "dyn": 8, "sync": 16, "own": 32, "swork": 64, "wring": 128, "tiny": 256, "coop": 512}

    def last_launch_path(self) -> set:
        """Execution path of this comm's last collective launch (test hook)."""
        f = _lib().mpxa__last_launch
        f.argtypes = [_P, ctypes.POINTER(ctypes.c_uint32)]
        f.restype = _I
        b = ctypes.c_uint32()
        _ck(f(self.handle, ctypes.byref(b)), "last_launch")
        return {k for k, v in self.PATH_BITS.items() if b.value & v}

    def check(self) -> int:
        return _lib().mpxa_comm_check(self.handle)

    def set_algorithm(self, op: str, algo):
        _ck(_lib().mpxa_set_algorithm(self.handle, OPS[op], _algo(algo)), "set_algorithm")

    def get_algorithm(self, op: str, nbytes: int) -> str:
        a = ctypes.c_int()
        _ck(_lib().mpxa_get_algorithm(self.handle, OPS[op], nbytes, ctypes.byref(a)), "get_algorithm")
        return ALGO_NAME[a.value]

    def config_digest(self) -> int:
        """Digest of the knobs / selector / forced variants compared across processes at init."""
        d = ctypes.c_uint64()
        _ck(_lib().mpxa_config_digest(self.handle, ctypes.byref(d)), "config_digest")
        return d.value

    def load_selector(self, path: str):
        _ck(_lib().mpxa_load_selector(self.handle, path.encode()), "load_selector")

    def register(self, t):
        _ck(_lib().mpxa_register(self.handle, _ptr(t), t.numel() * t.element_size()), "register")

    # ---- one-shot collectives ------------------------------------------------------
    def _count(self, send, per_rank_blocks: int) -> int:
        n = send.numel()
        d = self.R * per_rank_blocks
        if n % d:
            raise ValueError(f"send numel {n} not divisible by R*blocks = {d}")
        return n // d

    def alltoall(self, send, recv, algo=None, stream=None, count: Optional[int] = None):
        count = self._count(send, self.p) if count is None else count
        _ck(_lib().mpxa_alltoall_algo(_ptr(send), count, send.element_size(), _ptr(recv), _algo(algo),
                                      self.handle, _stream(stream)), "alltoall")

    def allgather(self, send, recv, algo=None, stream=None, count: Optional[int] = None):
        count = self._count(send, 1) if count is None else count
        _ck(_lib().mpxa_allgather_algo(_ptr(send), count, send.element_size(), _ptr(recv), _algo(algo),
                                       self.handle, _stream(stream)), "allgather")

    def alltoallv(self, send, sendcounts, sdispls, recv, recvcounts, rdispls, algo=None, stream=None,
                  dtype_size: Optional[int] = None):
        w = send.element_size() if dtype_size is None else dtype_size
        sc, scp = _i64_arg(sendcounts)
        sd, sdp = _i64_arg(sdispls)
        rc, rcp = _i64_arg(recvcounts)
        rd, rdp = _i64_arg(rdispls)
        sbpr = send.numel() * send.element_size() // self.R
        rbpr = recv.numel() * recv.element_size() // self.R
        _ck(_lib().mpxa_alltoallv_algo(_ptr(send), scp, sdp, sbpr, _ptr(recv), rcp, rdp, rbpr, w, _algo(algo),
                                       self.handle, _stream(stream)), "alltoallv")

    def alltoallv_counts(self, d_sendcounts, d_recvcounts, d_rdispls, stream=None):
        _ck(_lib().mpxa_alltoallv_counts(_ptr(d_sendcounts), _ptr(d_recvcounts), _ptr(d_rdispls),
                                         self.handle, _stream(stream)), "alltoallv_counts")

    def alltoall_bruck_stage(self, send, T, stage: int, stream=None):
        count = self._count(send, self.p)
        _ck(_lib().mpxa_alltoall_bruck_stage(_ptr(send), count, send.element_size(), _ptr(T), stage,
                                             self.handle, _stream(stream)), "alltoall_bruck_stage")

    def allgather_bruck_stage(self, send, T, stage: int, stream=None):
        count = self._count(send, 1)
        _ck(_lib().mpxa_allgather_bruck_stage(_ptr(send), count, send.element_size(), _ptr(T), stage,
                                              self.handle, _stream(stream)), "allgather_bruck_stage")

    # ---- persistent forms ---------------------------------------------------------
    def alltoall_init(self, send, recv, algo=None, count: Optional[int] = None) -> Request:
        count = self._count(send, self.p) if count is None else count
        h = ctypes.c_void_p()
        _ck(_lib().mpxa_alltoall_init(_ptr(send), count, send.element_size(), _ptr(recv), _algo(algo),
                                      self.handle, None, ctypes.byref(h)), "alltoall_init")
        return Request(self, h.value, (send, recv))

    def allgather_init(self, send, recv, algo=None, count: Optional[int] = None) -> Request:
        count = self._count(send, 1) if count is None else count
        h = ctypes.c_void_p()
        _ck(_lib().mpxa_allgather_init(_ptr(send), count, send.element_size(), _ptr(recv), _algo(algo),
                                       self.handle, None, ctypes.byref(h)), "allgather_init")
        return Request(self, h.value, (send, recv))

    def alltoallv_init(self, send, sendcounts, sdispls, recv, recvcounts, rdispls, algo=None,
                       dtype_size: Optional[int] = None) -> Request:
        w = send.element_size() if dtype_size is None else dtype_size
        arrs = [_i64_arg(a) for a in (sendcounts, sdispls, recvcounts, rdispls)]
        sbpr = send.numel() * send.element_size() // self.R
        rbpr = recv.numel() * recv.element_size() // self.R
        h = ctypes.c_void_p()
        _ck(_lib().mpxa_alltoallv_init(_ptr(send), arrs[0][1], arrs[1][1], sbpr, _ptr(recv), arrs[2][1],
                                       arrs[3][1], rbpr, w, _algo(algo), self.handle, None,
                                       ctypes.byref(h)), "alltoallv_init")
        return Request(self, h.value, (send, recv))

    # ---- neighborhood collectives --------------------------------
    def dist_graph_create_adjacent(self, sources, destinations, sourceweights=None, destweights=None,
                                   reorder: int = 0) -> "Topology":
        """sources / destinations: per local rank, the list of in / out neighbour ranks
        (MPIX_Dist_graph_create_adjacent).  Collective over the comm's processes."""
        indeg = np.array([len(x) for x in sources], np.int32)
        outdeg = np.array([len(x) for x in destinations], np.int32)
        if len(indeg) != self.R or len(outdeg) != self.R:
            raise ValueError(f"one neighbour list per local rank expected ({self.R})")
        src = np.array([v for x in sources for v in x], np.int32)
        dst = np.array([v for x in destinations for v in x], np.int32)
        sw = None if sourceweights is None else np.array([v for x in sourceweights for v in x], np.int32)
        dw = None if destweights is None else np.array([v for x in destweights for v in x], np.int32)
        h = ctypes.c_void_p()
        _ck(_lib().mpxa_dist_graph_create_adjacent(
            self.handle, indeg.ctypes.data, src.ctypes.data if len(src) else None,
            sw.ctypes.data if sw is not None and len(sw) else None, outdeg.ctypes.data,
            dst.ctypes.data if len(dst) else None, dw.ctypes.data if dw is not None and len(dw) else None,
            None, reorder, ctypes.byref(h)), "dist_graph_create_adjacent")
        return Topology(self, h.value)

    def _nb_args(self, send, sendcounts, sdispls, recv, recvcounts, rdispls, dtype_size):
        w = send.element_size() if dtype_size is None else dtype_size
        arrs = [_host_i64(a) for a in (sendcounts, sdispls, recvcounts, rdispls)]
        sbpr = send.numel() * send.element_size() // self.R
        rbpr = recv.numel() * recv.element_size() // self.R
        return w, arrs, sbpr, rbpr

    def neighbor_alltoallv_init(self, topo, send, sendcounts, sdispls, recv, recvcounts, rdispls,
                                dtype_size: Optional[int] = None, send_indices=None, recv_indices=None) -> Request:
        """Persistent neighbor alltoallv (counts / displacements: one entry per edge of the
        local ranks, rank-major); with send_indices / recv_indices (one global index per
        element) the locality-aware variant."""
        w, arrs, sbpr, rbpr = self._nb_args(send, sendcounts, sdispls, recv, recvcounts, rdispls, dtype_size)
        h = ctypes.c_void_p()
        if send_indices is None:
            _ck(_lib().mpxa_neighbor_alltoallv_init(
                _ptr(send), arrs[0][1], arrs[1][1], sbpr, _ptr(recv), arrs[2][1], arrs[3][1], rbpr, w,
                topo.handle, None, ctypes.byref(h)), "neighbor_alltoallv_init")
        else:
            si, sip = _host_i64(send_indices)
            ri, rip = _host_i64(recv_indices)
            _ck(_lib().mpxa_neighbor_alltoallv_locality_init(
                _ptr(send), arrs[0][1], arrs[1][1], sbpr, _ptr(recv), arrs[2][1], arrs[3][1], rbpr, w,
                sip, rip, topo.handle, None, ctypes.byref(h)), "neighbor_alltoallv_locality_init")
        return Request(self, h.value, (send, recv, topo))

    def neighbor_alltoallv(self, topo, send, sendcounts, sdispls, recv, recvcounts, rdispls, stream=None,
                           dtype_size: Optional[int] = None):
        w, arrs, sbpr, rbpr = self._nb_args(send, sendcounts, sdispls, recv, recvcounts, rdispls, dtype_size)
        _ck(_lib().mpxa_neighbor_alltoallv(_ptr(send), arrs[0][1], arrs[1][1], sbpr, _ptr(recv), arrs[2][1],
                                           arrs[3][1], rbpr, w, topo.handle, _stream(stream)), "neighbor_alltoallv")

    # ---- partitioned point-to-point ----------------------------------
    def psend_init(self, buf, partitions: int, rank: int, dest: int, tag: int = 0,
                   count: Optional[int] = None) -> "PRequest":
        """Partitioned send of `buf` (all of it, or `count` elements per partition) from local
        rank `rank` to `dest`; matched later by pmatch()."""
        count = buf.numel() // partitions if count is None else count
        h = ctypes.c_void_p()
        _ck(_lib().mpxa_psend_init(_ptr(buf), partitions, count, buf.element_size(), rank, dest, tag, self.handle,
                                   None, ctypes.byref(h)), "psend_init")
        return PRequest(self, h.value, buf, partitions, True)

    def precv_init(self, buf, partitions: int, rank: int, source: int, tag: int = 0,
                   count: Optional[int] = None) -> "PRequest":
        count = buf.numel() // partitions if count is None else count
        h = ctypes.c_void_p()
        _ck(_lib().mpxa_precv_init(_ptr(buf), partitions, count, buf.element_size(), rank, source, tag, self.handle,
                                   None, ctypes.byref(h)), "precv_init")
        return PRequest(self, h.value, buf, partitions, False)

    def pmatch(self):
        """The single match of every pending partitioned end (collective)."""
        _ck(_lib().mpxa_pmatch(self.handle), "pmatch")

    def finalize(self):
        if self.handle:
            _ck(_lib().mpxa_finalize(self.handle), "finalize")
            self.handle = None

    def __del__(self):
        try:
            if self.handle:
                _lib().mpxa_finalize(self.handle)
        except Exception:
            pass


class PRequest(Request):
    """One end of a partitioned channel (MPI-4 Psend_init / Precv_init)."""

    def __init__(self, comm, handle, buf, partitions, sender):
        super().__init__(comm, handle, buf)
        self.partitions = partitions
        self.sender = sender

    def pready(self, lo: int, hi: Optional[int] = None, stream=None):
        hi = lo + 1 if hi is None else hi
        _ck(_lib().mpxa_pready_range(self.handle, lo, hi, _stream(stream)), "pready")

    def parrived(self, j: int) -> bool:
        f = ctypes.c_int()
        _ck(_lib().mpxa_parrived(self.handle, j, ctypes.byref(f)), "parrived")
        return bool(f.value)

    def parrived_wait(self, lo: int, hi: Optional[int] = None, stream=None):
        hi = lo + 1 if hi is None else hi
        _ck(_lib().mpxa_parrived_wait(self.handle, lo, hi, _stream(stream)), "parrived_wait")

    def device_handle(self) -> bytes:
        """Bytes of the mpxa_psend_dev_t for mpxa_dev_pready in a user kernel."""
        buf = (ctypes.c_char * 128)()
        _ck(_lib().mpxa_psend_device(self.handle, buf, 128), "psend_device")
        return bytes(buf)


class Topology:
    """MPIX_Dist_graph_create_adjacent result."""

    def __init__(self, comm: Comm, handle: int):
        self.comm = comm
        self.handle = ctypes.c_void_p(handle)

    def free(self):
        if self.handle:
            h = ctypes.c_void_p(self.handle.value)
            _ck(_lib().mpxa_topo_free(ctypes.byref(h)), "topo_free")
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def make_bootstrap(group, nprocs: int):
    """A C callback doing the bootstrap all-gather over a gloo process group."""
    import torch
    import torch.distributed as dist

    def cb(inp, out, nbytes, ctx):
        try:
            src = torch.frombuffer(ctypes.string_at(inp, nbytes), dtype=torch.uint8).clone() if nbytes else \
                torch.empty(0, dtype=torch.uint8)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(nprocs)]
            dist.all_gather(outs, src, group=group)
            buf = torch.cat(outs).numpy().tobytes()
            ctypes.memmove(out, buf, len(buf))
            return 0
        except Exception:   # the library maps a non-zero return to an error status
            return 1

    return BOOT_FN(cb)


# ---- host-only plan introspection (no GPU needed) ---------------------------------------
class Plan:
    """A compiled schedule (include/mpxa_plan.h), for CPU simulation in tests."""

    def __init__(self, op: str, algo: str, p: int, R: int = 0, G: int = 1, g: int = 1, stop_stage: int = -1,
                 counts=None, sdispls=None, rdispls=None):
        R = R or p // G
        h = ctypes.c_void_p()
        keep = []
        cp = sp = rp = None
        if counts is not None:
            (c, cp), (s, sp), (r, rp) = _host_i64(counts), _host_i64(sdispls), _host_i64(rdispls)
            keep = [c, s, r]
        _ck(_lib().mpxa_plan_build(OPS[op], ALGO[algo], p, R, G, g, stop_stage, cp, sp, rp, ctypes.byref(h)),
            "plan_build")
        self.h = h
        self.p, self.R, self.G = p, R, G
        self._keep = keep
        info = PlanInfo()
        _ck(_lib().mpxa_plan_info(h, ctypes.byref(info)), "plan_info")
        self.info = {n: int(getattr(info, n)) for n, _ in PlanInfo._fields_}

    @classmethod
    def neighbor(cls, gr, R: int, G: int, g: int = 1, locality: bool = False, send_idx=None, recv_idx=None):
        """Schedule of a neighbor alltoallv over a GLOBAL graph dict (oracle/synth layout)."""
        self = cls.__new__(cls)
        p = len(gr["indeg"])
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        arrs = [i32(gr["indeg"]), i32(gr["src"]), np.ascontiguousarray(gr["rc"], np.int64),
                np.ascontiguousarray(gr["rd"], np.int64), i32(gr["outdeg"]), i32(gr["dst"]),
                np.ascontiguousarray(gr["sc"], np.int64), np.ascontiguousarray(gr["sd"], np.int64)]
        si = np.ascontiguousarray(send_idx, np.int64) if send_idx is not None else None
        ri = np.ascontiguousarray(recv_idx, np.int64) if recv_idx is not None else None
        h = ctypes.c_void_p()
        ptr = lambda a: a.ctypes.data if a is not None and a.size else None
        _ck(_lib().mpxa_plan_build_neighbor(p, R, G, g, int(locality), *[ptr(a) for a in arrs], ptr(si), ptr(ri),
                                            ctypes.byref(h)), "plan_build_neighbor")
        self.h = h
        self.p, self.R, self.G = p, R, G
        self._keep = arrs + [si, ri]
        info = PlanInfo()
        _ck(_lib().mpxa_plan_info(h, ctypes.byref(info)), "plan_info")
        self.info = {n: int(getattr(info, n)) for n, _ in PlanInfo._fields_}
        return self

    def eager(self, unit: int) -> "Plan":
        """The eager (LL) form of this multi-GPU plan for `unit` bytes per unit
        (mpxa_plan_eager): raises MpxaError(ERR_ALGO) when ineligible."""
        h = ctypes.c_void_p()
        _ck(_lib().mpxa_plan_eager(self.h, unit, ctypes.byref(h)), "plan_eager")
        q = Plan.__new__(Plan)
        q.h = h
        q.p, q.R, q.G = self.p, self.R, self.G
        q._keep = []
        info = PlanInfo()
        _ck(_lib().mpxa_plan_info(h, ctypes.byref(info)), "plan_info")
        q.info = {n: int(getattr(info, n)) for n, _ in PlanInfo._fields_}
        return q

    def steps(self, gpu: int):
        n = ctypes.c_int(0)
        _ck(_lib().mpxa_plan_steps(self.h, gpu, None, ctypes.byref(n)), "plan_steps")
        arr = (PlanStep * max(1, n.value))()
        _ck(_lib().mpxa_plan_steps(self.h, gpu, arr, ctypes.byref(n)), "plan_steps")
        return [arr[i] for i in range(n.value)]

    def moves(self, gpu: int):
        n = ctypes.c_int(0)
        _ck(_lib().mpxa_plan_moves(self.h, gpu, None, ctypes.byref(n)), "plan_moves")
        arr = (PlanMove * max(1, n.value))()
        _ck(_lib().mpxa_plan_moves(self.h, gpu, arr, ctypes.byref(n)), "plan_moves")
        return [arr[i] for i in range(n.value)]

    def __del__(self):
        try:
            if self.h:
                _lib().mpxa_plan_free(self.h)
        except Exception:
            pass

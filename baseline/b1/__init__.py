"""B1: NCCL grouped send/recv and all-gather from C++ (BASELINE.md §4.1).

The baseline the paper's collectives are layered over (MPI Advance sits on
the system MPI; on B200 the system library is NCCL).  libnccl_b1.so wraps NCCL 2.28 (the
torch-bundled library) behind a tiny C ABI; timing loops and CUDA-graph capture run in C++
(baseline/b1/nccl_b1.cpp), Python only exchanges the unique id and marshals pointers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "nccl_b1.cpp")
LIB = os.path.join(HERE, "libnccl_b1.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

OPS = {"alltoall": 0, "allgather": 1, "allgather_grouped": 2, "alltoallv": 3}


def nccl_dir() -> str:
    import nvidia.nccl
    return list(nvidia.nccl.__path__)[0]


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    nd = nccl_dir()
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC",
                           "-I" + os.path.join(nd, "include"), SRC, "-o", tmp,
                           "-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2",
                           "-Xlinker", "-rpath=" + os.path.join(nd, "lib")])
    os.replace(tmp, LIB)
    return LIB


_L = None


def lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built (baseline.b1.build())")
        L = ctypes.CDLL(LIB)
        P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        L.b1_version.argtypes = [ctypes.POINTER(I)]
        L.b1_unique_id.argtypes = [P, Z]
        L.b1_init.argtypes = [ctypes.POINTER(P), I, I, P, I]
        L.b1_finalize.argtypes = [P]
        L.b1_call.argtypes = [P, I, P, P, Z, P, P, P, P, P]
        L.b1_time.argtypes = [P, I, P, P, Z, P, P, P, P, P, I, I, I, ctypes.POINTER(ctypes.c_double)]
        for f in (L.b1_version, L.b1_unique_id, L.b1_init, L.b1_finalize, L.b1_call, L.b1_time):
            f.restype = I
        _L = L
    return _L


def version() -> str:
    v = ctypes.c_int()
    assert lib().b1_version(ctypes.byref(v)) == 0
    x = v.value
    return f"{x // 10000}.{(x // 100) % 100}.{x % 100}"


def _ck(rc, what):
    if rc:
        raise RuntimeError(f"B1 {what} failed: code {rc}")


class NcclB1:
    """One NCCL communicator over the processes of `pg` (one rank per GPU)."""

    def __init__(self, pg, device: int):
        import torch.distributed as dist
        self.n, self.rank = dist.get_world_size(pg), dist.get_rank(pg)
        idbuf = (ctypes.c_char * 128)()
        if self.rank == 0:
            _ck(lib().b1_unique_id(idbuf, 128), "unique_id")
        obj = [bytes(idbuf)]
        dist.broadcast_object_list(obj, src=0, group=pg)
        idbuf = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        self.h = ctypes.c_void_p()
        _ck(lib().b1_init(ctypes.byref(self.h), self.n, self.rank, idbuf, device), "init")

    @staticmethod
    def _v(arrs):
        import numpy as np
        if arrs is None:
            return [None] * 4, []
        keep = [np.ascontiguousarray(a, dtype=np.int64) for a in arrs]
        return [k.ctypes.data_as(ctypes.c_void_p) for k in keep], keep

    def call(self, op, send, recv, nbytes=0, v=None, stream=None):
        ptrs, keep = self._v(v)
        _ck(lib().b1_call(self.h, OPS[op], send.data_ptr(), recv.data_ptr(), nbytes, *ptrs,
                          _stream(stream)), op)

    def time(self, op, send, recv, nbytes=0, v=None, stream=None, warmup=5, iters=20, graph=False) -> float:
        ptrs, keep = self._v(v)
        us = ctypes.c_double()
        _ck(lib().b1_time(self.h, OPS[op], send.data_ptr(), recv.data_ptr(), nbytes, *ptrs, _stream(stream),
                          warmup, iters, int(graph), ctypes.byref(us)), op + " timing")
        return us.value

    def finalize(self):
        if self.h:
            lib().b1_finalize(self.h)
            self.h = None


def _stream(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream

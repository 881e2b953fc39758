"""B200-native GPU-resident alltoall / alltoallv / allgather (MPI Advance, arXiv 2309.07337).

The product is libmpxa.so (C ABI in include/mpxa.h; sm_100a kernels in csrc/); this
package is its thin ctypes binding.  See DESIGN.md.
"""
from .mpxa import (ALGO, ALGO_NAME, OPS, Comm, MpxaError, Plan, PRequest, Request, Topology, lib,  # noqa: F401
                   list_algorithms)

__all__ = ["Comm", "Request", "Plan", "MpxaError", "list_algorithms", "lib", "ALGO", "OPS"]

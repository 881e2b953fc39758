"""Per-CTA timeline of ONE single-GPU allgather launch inside a back-to-back CUDA graph (p = 8;
MPXA_TRACE build, MPXA_LIB=<libmpxa_trace.so>): CTA entry, return from the dependency wait
(griddepcontrol), first queue piece taken, exit -- percentiles in us from the earliest entry,
next to the graph-timed us per call.  Where a launch's time goes beyond HBM streaming."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
from paper_2309_07337_b200 import Comm, lib
from timing import t
L = lib()
L.mpxa__cta_trace.argtypes = [ctypes.c_void_p]
p = 8
c = Comm(ranks_per_proc=p, device=0)
big = torch.randint(0, 255, (p * (64 << 20),), dtype=torch.uint8, device="cuda")
for b in [int(x) << 20 for x in os.environ.get("SIZES_MIB", "4,8,64").split(",")]:
    s = big[: p * b].view(p, b)
    r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
    L.mpxa__cta_trace(None)
    us = t(lambda: c.allgather(s, r), it=10)     # the last launch of the last replay stays recorded
    buf = (ctypes.c_uint64 * 6144)()
    L.mpxa__cta_trace(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(6, 1024).astype(np.int64)
    n = int((a[0] > 0).sum())
    t0 = a[0, :n].min()
    q = lambda x: [round(float(np.percentile(x - t0, v)) / 1e3, 2) for v in (0, 10, 50, 90, 100)]
    print(b >> 20, "MiB graph us/call", round(us, 1), sorted(c.last_launch_path()), "ctas", n,
          "entry", q(a[0, :n]), "after_wait", q(a[2, :n]), "classified", q(a[4, :n]), "first_piece", q(a[3, :n]), "first_store", q(a[5, :n]), "exit", q(a[1, :n]), flush=True)
    del r

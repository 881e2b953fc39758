"""Per-CTA timeline of one cfg4 alltoallv launch (p = 8, persistent start+wait in a back-to-back
CUDA graph; MPXA_TRACE build via MPXA_LIB): CTA entry, return from the dependency wait, tile
classified, warp 0's first stage landed, exit -- percentiles in us from the earliest entry."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import synth
import timing
from paper_2309_07337_b200 import Comm, lib
from timing import t
L = lib()
L.mpxa__cta_trace.argtypes = [ctypes.c_void_p]
p = 8
c = Comm(ranks_per_proc=p, device=0)
for mean in (float(x) for x in os.environ.get("MEANS", "1,4").split(",")):
    c4 = synth.cfg4_counts(0, p, int(mean * (1 << 20)), elem=8)
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c4, elem=8)
    d_s = torch.from_numpy(send).cuda()
    d_r = torch.zeros((p, Rcap), dtype=torch.uint8, device="cuda")
    q = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, dtype_size=8)
    L.mpxa__cta_trace(None)
    us = t(lambda: (q.start(timing.GS), q.wait(timing.GS)), it=10)
    buf = (ctypes.c_uint64 * 6144)()
    L.mpxa__cta_trace(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(6, 1024).astype(np.int64)
    n = int((a[0] > 0).sum())
    t0 = a[0, :n].min()
    qq = lambda x: [round(float(np.percentile(x - t0, v)) / 1e3, 2) for v in (0, 10, 50, 90, 100)]
    print(mean, "MiB mean, graph us/call", round(us, 1), sorted(c.last_launch_path()), "ctas", n,
          "entry", qq(a[0, :n]), "after_wait", qq(a[2, :n]), "tile", qq(a[4, :n]), "first_stage", qq(a[5, :n]),
          "exit", qq(a[1, :n]), flush=True)
    q.free()

"""Phase stamps (SM cycles, clock64) of CTA 0 (producer thread 0 / LSU thread 32) for one
launch (MPXA_TRACE build: MPXA_LIB=.../libmpxa_trace.so), next to the device time per call
of the same launch in a CUDA graph.  CASES="op:bytes,..." """
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm, lib
L = lib(); f = L.mpxa__trace; f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]; f.restype = ctypes.c_int
p = int(os.environ.get("P", "8"))
c = Comm(ranks_per_proc=p, device=0, emulate_gpus=int(os.environ.get("EMU", "0")))
GS = torch.cuda.Stream()
cases = os.environ.get("CASES", "allgather:4,alltoall:4,allgather:1024,alltoall:16384,allgather:16384,alltoall:65536,alltoall:1048576")
for case in cases.split(","):
    op, b = case.split(":"); b = int(b)
    if op == "allgather":
        s = torch.zeros((p, b), dtype=torch.uint8, device="cuda"); r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
        fn = lambda: c.allgather(s, r, algo=os.environ.get("ALGO", "pairwise"), stream=GS)
    else:
        s = torch.zeros((p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
        fn = lambda: c.alltoall(s, r, algo=os.environ.get("ALGO", "pairwise"), stream=GS)
    for _ in range(5): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=GS):
        for _ in range(20): fn()
    with torch.cuda.stream(GS):
        g.replay(); torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(GS); g.replay(); e.record(GS); torch.cuda.synchronize()
    us = a.elapsed_time(e) / 20 * 1e3
    buf = (ctypes.c_uint64 * 32)()
    f(c.handle, buf)
    t0 = buf[0]
    print(op, b, f"graph us/call={us:.2f}", "producer:", [int(buf[i] - t0) if buf[i] else None for i in range(16)],
          "lsu warp1:", [int(buf[16 + i] - t0) if buf[16 + i] else None for i in range(9)], flush=True)
# per-CTA entry/exit of the last launch (exec kernel): spread of starts and ends
if hasattr(L, "mpxa__cta_trace"):
    import numpy as np
    for case in os.environ.get("CTA_CASES", "alltoall:1048576,alltoall:4194304,allgather:1048576").split(","):
        op, b = case.split(":"); b = int(b)
        if op == "allgather":
            s = torch.zeros((p, b), dtype=torch.uint8, device="cuda"); r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
            fn = lambda: c.allgather(s, r, algo=os.environ.get("ALGO", "pairwise"), stream=GS)
        else:
            s = torch.zeros((p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
            fn = lambda: c.alltoall(s, r, algo=os.environ.get("ALGO", "pairwise"), stream=GS)
        buf = (ctypes.c_uint64 * 2048)()
        for _ in range(4): fn()
        torch.cuda.synchronize()
        ctypes.memset(buf, 0, 2048 * 8)
        L.mpxa__cta_trace.argtypes = [ctypes.c_void_p]
        torch.cuda.synchronize(); L.mpxa__cta_trace(None)   # clear, run one launch, read
        fn(); torch.cuda.synchronize()
        L.mpxa__cta_trace(buf)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024).astype(np.int64)
        n = int((a[0] > 0).sum())
        st, en = a[0, :n], a[1, :n]
        t0 = st.min()
        q = lambda x: [int(np.percentile(x - t0, v)) for v in (0, 50, 90, 100)]
        d = en - st
        print(op, b, "ctas", n, "dur min/p50/max", int(d.min()), int(np.median(d)), int(d.max()), "start p0/50/90/100", q(st), "end", q(en), "dur p50", int(np.median(en - st)), flush=True)

"""Time the hot workloads for one libmpxa build (MPXA_LIB selects a tuning variant)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm

import time
GS = torch.cuda.Stream()

def t(fn, it=20, w=3):
    """device us per call: `it` calls captured in a CUDA graph, median of 3 replays"""
    for _ in range(w): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=GS):
        for _ in range(it): fn()
    ts = []
    with torch.cuda.stream(GS):
        g.replay(); torch.cuda.synchronize()
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(GS); g.replay(); b.record(GS); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / it * 1e3)
    return sorted(ts)[1]

p = 8
c = Comm(ranks_per_proc=p, device=0)
res = {"lib": os.path.basename(os.environ.get("MPXA_LIB", "libmpxa.so")), "ns": os.environ.get("MPXA_NS"), "nf": os.environ.get("MPXA_NF")}
for b in (64 << 20, 4 << 20, 1 << 20):
    s = torch.randint(0, 255, (p, b), dtype=torch.uint8, device="cuda")
    r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
    us = t(lambda: c.allgather(s, r, algo="pairwise", stream=GS))
    res[f"ag_{b>>20}M_us"] = round(us, 1); res[f"ag_{b>>20}M_hbm_tbs"] = round((p * b + p * p * b) / us / 1e6, 3)
    del s, r
for b in (16 << 20, 1 << 20):
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
    r = torch.empty_like(s)
    us = t(lambda: c.alltoall(s, r, algo="pairwise", stream=GS))
    res[f"a2a_{b>>20}M_us"] = round(us, 1); res[f"a2a_{b>>20}M_hbm_tbs"] = round(2 * p * p * b / us / 1e6, 3)
    del s, r
# small messages: device latency (graph) and host submission cost (wall clock per call)
for b in (4, 4096):
    s = torch.zeros((p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
    for algo in ("pairwise", "bruck"):
        res[f"a2a_{b}B_{algo}_us"] = round(t(lambda: c.alltoall(s, r, algo=algo, stream=GS), it=50), 2)
    s2 = torch.zeros((p, b), dtype=torch.uint8, device="cuda"); r2 = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
    res[f"ag_{b}B_us"] = round(t(lambda: c.allgather(s2, r2, algo="pairwise", stream=GS), it=50), 2)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(200): c.alltoall(s, r, algo="pairwise", stream=GS)
    res[f"host_submit_us_per_call_{b}B"] = round((time.perf_counter() - h0) / 200 * 1e6, 2)
    torch.cuda.synchronize()
if os.environ.get("COPY_REF"):
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda"); bb = torch.empty_like(a)
    us = t(lambda: bb.copy_(a)); res["torch_copy_1G_tbs"] = round(2 * (1 << 30) / us / 1e6, 3)
    a2 = torch.empty(4 << 30, dtype=torch.uint8, device="cuda"); s2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    us = t(lambda: a2.view(8, -1).copy_(s2.view(1, -1).expand(8, -1)))
    res["torch_bcast_512M_x8_tbs"] = round((4.5 * (1 << 30)) / us / 1e6, 3)
print(json.dumps(res), flush=True)

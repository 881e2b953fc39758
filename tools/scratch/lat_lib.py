"""Per-call device latency (graph) of tiny collectives through libmpxa, by p."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
GS = torch.cuda.Stream()
def t(fn, it=50):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=GS):
        for _ in range(it): fn()
    with torch.cuda.stream(GS):
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(GS); g.replay(); b.record(GS); torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3
for p in (1, 2, 4, 8, 16):
    c = Comm(ranks_per_proc=p, device=0)
    s = torch.zeros((p, p * 4), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
    print(p, {a: round(t(lambda: c.alltoall(s, r, algo=a, stream=GS)), 2) for a in ("pairwise", "bruck")}, flush=True)

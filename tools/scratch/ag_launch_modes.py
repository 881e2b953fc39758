"""allgather p = 8, 4 / 8 MiB: graph-timed vs a plain stream loop (20 launches between events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
from timing import t
p = 8
c = Comm(ranks_per_proc=p, device=0)
big = torch.randint(0, 255, (p * (8 << 20),), dtype=torch.uint8, device="cuda")
for b in (4 << 20, 8 << 20):
    s = big[: p * b].view(p, b)
    r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
    g = t(lambda: c.allgather(s, r), it=20)
    for _ in range(3): c.allgather(s, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): c.allgather(s, r)
    e1.record(); torch.cuda.synchronize()
    print(b >> 20, "MiB graph", round(g, 1), "plain", round(e0.elapsed_time(e1) * 1e3 / 20, 1), os.environ.get("MPXA_NO_PDL", ""), flush=True)

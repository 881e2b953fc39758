"""Multi-step small launches on one GPU (p = 8): Bruck / hierarchical alltoall and Bruck / ring
allgather, device us per call (CUDA graph of 200 calls) and path, with the tiny multi-step
kernel and with MPXA_NO_TINY=1."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2309_07337_b200 import Comm
from timing import t
res = {}
for knob in ("", "MPXA_NO_TINY"):
    if knob:
        os.environ[knob] = "1"
    c = Comm(ranks_per_proc=8, device=0)
    if knob:
        del os.environ[knob]
    for b in (16, 256, 4096):
        s = torch.randint(0, 255, (8, 8 * b), dtype=torch.uint8, device="cuda")
        r = torch.empty_like(s)
        for algo in ("bruck", "hier"):
            us = t(lambda: c.alltoall(s, r, algo=algo), it=200)
            res[f"{knob or 'tiny'}_a2a_{algo}_{b}"] = [round(us, 3), sorted(c.last_launch_path())]
        s2 = s[:, :b].contiguous()
        for algo in ("bruck", "ring"):
            us = t(lambda: c.allgather(s2, r, algo=algo), it=200)
            res[f"{knob or 'tiny'}_ag_{algo}_{b}"] = [round(us, 3), sorted(c.last_launch_path())]
    c.finalize()
print(json.dumps(res))

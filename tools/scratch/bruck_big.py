"""Bruck / ring at large blocks on one GPU (p = 8): device us and the launch path."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
p = 8
c = Comm(ranks_per_proc=p, device=0)
res = {}
for b in (1 << 20, 4 << 20):
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
    for algo in ("bruck",):
        us = t(lambda: c.alltoall(s, r, algo=algo, stream=GS), it=5)
        res[f"a2a_{algo}_{b>>20}M"] = [round(us, 1), sorted(c.last_launch_path())]
    s2 = s[:, :b].contiguous()
    for algo in ("bruck", "ring"):
        us = t(lambda: c.allgather(s2, r, algo=algo, stream=GS), it=5)
        res[f"ag_{algo}_{b>>20}M"] = [round(us, 1), sorted(c.last_launch_path())]
print(json.dumps(res))

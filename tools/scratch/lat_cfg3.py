"""cfg3-shaped tiny alltoalls (float32 payload, p = 2 / 4 ranks on one GPU) and cfg1
(p = 4, 8 int32): device us per call in CUDA graphs.  One JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
res = {}
for p in (2, 4):
    c = Comm(ranks_per_proc=p, device=0)
    for b in (4, 16, 64, 256, 1024):
        s = torch.rand((p, p * b // 4), dtype=torch.float32, device="cuda")
        r = torch.empty_like(s)
        for algo in ("pairwise", "bruck"):
            res[f"p{p}_{algo}_{b}"] = round(t(lambda: c.alltoall(s, r, algo=algo, stream=GS), it=20), 2)
    c.finalize()
c = Comm(ranks_per_proc=4, device=0)
s = torch.randint(0, 1 << 30, (4, 32), dtype=torch.int32, device="cuda"); r = torch.empty_like(s)
for algo in ("pairwise", "bruck"):
    res[f"cfg1_{algo}"] = round(t(lambda: c.alltoall(s, r, algo=algo, stream=GS), it=20), 2)
print(json.dumps(res), flush=True)

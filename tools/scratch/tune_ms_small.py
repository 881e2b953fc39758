"""Multi-step variants at small / mid sizes on one GPU (p=8), device us per call (graphs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
p = 8
res = {"no_small_sync": os.environ.get("MPXA_NO_SMALL_SYNC", "0")}
c = Comm(ranks_per_proc=p, device=0)
c2 = Comm(ranks_per_proc=p, device=0, group_size=2)
for b in (1024, 4096, 16384, 65536):
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
    res[f"a2a_bruck_{b}"] = round(t(lambda: c.alltoall(s, r, algo="bruck", stream=GS)), 2)
    res[f"a2a_hier2_{b}"] = round(t(lambda: c2.alltoall(s, r, algo="hier", stream=GS)), 2)
    s2 = s[:, :b].contiguous()
    res[f"ag_ring_{b}"] = round(t(lambda: c.allgather(s2, r, algo="ring", stream=GS)), 2)
    res[f"ag_bruck_{b}"] = round(t(lambda: c.allgather(s2, r, algo="bruck", stream=GS)), 2)
counts = synth.cfg4_counts(0, p, 65536)
sc = counts.astype(np.int64); rc = counts.T.copy()
sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
s_ = torch.randint(0, 255, (p, int((sd + sc).max()) * 8), dtype=torch.uint8, device="cuda")
r_ = torch.zeros((p, int((rd + rc).max()) * 8), dtype=torch.uint8, device="cuda")
for algo in ("hier", "bruck"):
    q = c2.alltoallv_init(s_, sc, sd, r_, rc, rd, dtype_size=8, algo=algo)
    res[f"a2av64K_{algo}"] = round(t(lambda: (q.start(GS), q.wait(GS))), 2)
    q.free()
print(json.dumps(res), flush=True)

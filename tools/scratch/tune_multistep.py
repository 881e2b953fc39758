"""Multi-step variants on one GPU (p=8): Bruck / hierarchical alltoall, ring / Bruck allgather,
device us per call in CUDA graphs (MPXA_NO_DYN=1 for the static executor)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t

tune_mid.GS = GS = torch.cuda.Stream()
p = 8
res = {"nodyn": os.environ.get("MPXA_NO_DYN", "0")}
c = Comm(ranks_per_proc=p, device=0)
c2 = Comm(ranks_per_proc=p, device=0, group_size=2)
for b in (1 << 20, 4 << 20, 16 << 20):
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
    r = torch.empty_like(s)
    res[f"a2a_bruck_{b >> 20}M"] = round(t(lambda: c.alltoall(s, r, algo="bruck", stream=GS), it=5), 1)
    res[f"a2a_hier2_{b >> 20}M"] = round(t(lambda: c2.alltoall(s, r, algo="hier", stream=GS), it=5), 1)
    s2 = s[:, :b].contiguous()
    res[f"ag_ring_{b >> 20}M"] = round(t(lambda: c.allgather(s2, r, algo="ring", stream=GS), it=5), 1)
    res[f"ag_bruck_{b >> 20}M"] = round(t(lambda: c.allgather(s2, r, algo="bruck", stream=GS), it=5), 1)
    del s, r
print(json.dumps(res), flush=True)

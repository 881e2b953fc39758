"""alltoall / allgather with many ranks on one GPU (p = 16, 32: more moves than one tile)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
from tune_mid import t  # noqa: E402  (graph timing helper)
GS = torch.cuda.Stream()
res = {"nodyn": os.environ.get("MPXA_NO_DYN", "0")}
for p in (16, 32):
    c = Comm(ranks_per_proc=p, device=0)
    for b in (65536, 262144, 1 << 20):
        s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
        r = torch.empty_like(s)
        import tune_mid
        tune_mid.GS = GS
        us = t(lambda: c.alltoall(s, r, algo="pairwise", stream=GS))
        res[f"a2a_p{p}_{b >> 10}K"] = [round(us, 1), round(2 * p * p * b / us / 1e6, 2)]
        del s, r
    c.finalize()
print(json.dumps(res), flush=True)

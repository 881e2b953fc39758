"""Mid-size latency probe (device us per call, CUDA graphs; SIZES / PS / EMU env): alltoall
and allgather variants.  One JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
res = {}
for p in [int(x) for x in os.environ.get("PS", "8").split(",")]:
    c = Comm(ranks_per_proc=p, device=0, emulate_gpus=int(os.environ.get("EMU", "0")))
    for b in [int(x) for x in os.environ.get("SIZES", "65536,262144,1048576,4194304").split(",")]:
        s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
        r = torch.empty_like(s)
        for algo in ("pairwise", "bruck", "hier"):
            res[f"a2a_p{p}_{algo}_{b}"] = round(t(lambda: c.alltoall(s, r, algo=algo, stream=GS), it=20), 2)
        s2 = s[:, :b].contiguous()
        for algo in ("pairwise", "bruck", "ring"):
            res[f"ag_p{p}_{algo}_{b}"] = round(t(lambda: c.allgather(s2, r, algo=algo, stream=GS), it=20), 2)
    c.finalize()
print(json.dumps(res), flush=True)

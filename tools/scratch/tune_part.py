"""Partitioned channel cycle timing on one GPU (CUDA graph): both starts, Pready of all, waits."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
c = Comm(ranks_per_proc=2, device=0)
res = {}
for nbytes, n_s, n_r in ((4096, 1, 1), (1 << 20, 4, 2), (64 << 20, 16, 4)):
    sb = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda"); rb = torch.zeros_like(sb)
    ps = c.psend_init(sb, n_s, 0, 1); pr = c.precv_init(rb, n_r, 1, 0); c.pmatch()
    def cyc():
        pr.start(GS); ps.start(GS); ps.pready(0, n_s, stream=GS); ps.wait(GS); pr.wait(GS)
    res[f"{nbytes}"] = round(t(cyc, it=20), 2)
    torch.cuda.synchronize()
    res[f"{nbytes}_ok"] = bool(torch.equal(sb, rb))
    ps.free(); pr.free()
print(json.dumps(res))

"""cfg4 alltoallv (p = 8, mean 4 MiB) with 8-byte elements vs the same bytes as 16-byte
elements (every segment 16-B congruent -> all TMA): persistent, device us in a CUDA graph."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
p = 8
c = Comm(ranks_per_proc=p, device=0)
res = {}
for elem in (8, 16):
    c4 = synth.cfg4_counts(0, p, 4 << 20)
    if elem == 16:
        c4 = c4 // 2   # same bytes
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c4, elem=elem)
    d_s = torch.from_numpy(send).cuda(); d_r = torch.zeros((p, Rcap), dtype=torch.uint8, device="cuda")
    q = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, dtype_size=elem)
    us = t(lambda: (q.start(GS), q.wait(GS)), it=10)
    moved = int(sc.sum()) * elem
    res[f"elem{elem}"] = [round(us, 1), round(2 * moved / us / 1e6, 2), sorted(c.last_launch_path())]
    q.free()
print(json.dumps(res))

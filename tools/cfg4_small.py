"""cfg4 alltoallv at mean 64 B and 64 KiB (p = 8, int64, persistent, CUDA graph): device us and
execution path, for int64 elements vs the same bytes as 16-byte elements."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import synth
from paper_2309_07337_b200 import Comm
from timing import t, GS
p = 8
knobs = dict(kv.split("=") for kv in os.environ.get("KNOBS", "").split(",") if kv)
for k, v in knobs.items():
    os.environ[k] = v
c = Comm(ranks_per_proc=p, device=0)
res = {"knobs": knobs}
for mean in [int(x) for x in os.environ.get("MEANS", "64,4096,65536,1048576").split(",")]:
    for elem in (8, 16):
        c4 = synth.cfg4_counts(0, p, mean, elem=8)
        if elem == 16:
            c4 = (c4 + 1) // 2
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c4, elem=elem)
        d_s = torch.from_numpy(send).cuda()
        d_r = torch.zeros((p, Rcap), dtype=torch.uint8, device="cuda")
        q = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, dtype_size=elem, algo="pairwise")
        us = t(lambda: (q.start(GS), q.wait(GS)), it=50)
        res[f"mean{mean}_elem{elem}"] = [round(us, 2), sorted(c.last_launch_path())]
        q.free()
print(json.dumps(res))

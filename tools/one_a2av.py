"""One cfg4-shaped alltoallv (p=8, mean MEAN bytes, int64) for profiling: 6 persistent cycles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2309_07337_b200 import Comm
p = 8
mean = int(os.environ.get("MEAN", str(4 << 20)))
c = Comm(ranks_per_proc=p, device=0)
counts = synth.cfg4_counts(0, p, mean)
sc = counts.astype(np.int64); rc = counts.T.copy()
sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
S = int((sd + sc).max()) * 8; R = int((rd + rc).max()) * 8
s = torch.randint(0, 255, (p, S), dtype=torch.uint8, device="cuda")
r = torch.zeros((p, R), dtype=torch.uint8, device="cuda")
q = c.alltoallv_init(s, sc, sd, r, rc, rd, dtype_size=8)
for _ in range(6):
    q.start(); q.wait()
torch.cuda.synchronize()
print("ok")

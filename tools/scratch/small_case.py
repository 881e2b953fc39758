"""Tiny alltoall / allgather launches for latency profiling (ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
p = 8
c = Comm(ranks_per_proc=p, device=0)
b = int(os.environ.get("B", "4"))
s = torch.zeros((p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
for _ in range(8):
    c.alltoall(s, r, algo=os.environ.get("ALGO", "pairwise"))
torch.cuda.synchronize()
print("ok")

"""A few p=8 alltoall launches at one block size (for ncu A/B captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
p = 8
b = int(os.environ.get("B", str(16 << 20)))
c = Comm(ranks_per_proc=p, device=0, emulate_gpus=int(os.environ.get("EMU", "0")))
s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
for _ in range(5):
    c.alltoall(s, r, algo=os.environ.get("ALGO", "pairwise"))
torch.cuda.synchronize()
print("ok")

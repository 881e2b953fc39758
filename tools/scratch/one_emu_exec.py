"""A few emulated-GPU executor launches (p = 32 on 8 virtual GPUs, 64 KiB blocks, executor
forced) for ncu captures."""
import os, sys
os.environ.setdefault("MPXA_NO_SMALL", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
p, G, b = 32, int(os.environ.get("EMU", "8")), int(os.environ.get("B", "65536"))
c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G)
s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
for _ in range(5):
    c.alltoall(s, r, algo="pairwise")
torch.cuda.synchronize()
print("ok")

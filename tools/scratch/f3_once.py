"""A few plain (non-graph) f3 cycles for an ncu launch list: SIZE_MIB, NS, NR from the env."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2309_07337_b200 import Comm
c = Comm(ranks_per_proc=2, device=0)
nbytes = int(float(os.environ.get("SIZE_MIB", "1")) * (1 << 20))
n_s, n_r = int(os.environ.get("NS", "4")), int(os.environ.get("NR", "2"))
sb = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda")
rb = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
ps = c.psend_init(sb, n_s, 0, 1)
pr = c.precv_init(rb, n_r, 1, 0)
c.pmatch()
for _ in range(3):
    pr.start(); ps.start(); ps.pready(0, n_s); ps.wait(); pr.wait()
torch.cuda.synchronize()
print("verified", bool(torch.equal(rb, sb)))

"""f3 partitioned channel on one GPU (rank 0 -> rank 1): CUDA-graph timed whole cycles, verified."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
from timing import t, GS
c = Comm(ranks_per_proc=2, device=0)
for nbytes, n_s, n_r in ((4096, 1, 1), (1 << 20, 4, 2), (16 << 20, 16, 4), (256 << 20, 16, 4), (256 << 20, 4, 16)):
    with torch.cuda.stream(GS):
        sb = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda")
        rb = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    ps = c.psend_init(sb, n_s, 0, 1)
    pr = c.precv_init(rb, n_r, 1, 0)
    c.pmatch()
    def cycle():
        pr.start(GS); ps.start(GS)
        ps.pready(0, n_s, stream=GS)
        ps.wait(GS); pr.wait(GS)
    us = t(cycle, it=10)
    torch.cuda.synchronize()
    print(nbytes >> 10, "KiB", f"{n_s}->{n_r}", round(us, 2), "us", round(2 * nbytes / us / 1e3, 1), "GB/s HBM",
          "verified", bool(torch.equal(rb, sb)), flush=True)
    ps.free(); pr.free()
c.finalize()

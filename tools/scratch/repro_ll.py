"""Find the first failing (p, b, G, algo) of the alltoall sweep, one launch at a time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import synth, oracle
from paper_2309_07337_b200 import Comm
p = int(os.environ.get("P", "8"))
for G in [int(x) for x in os.environ.get("GS", "2,4,8").split(",")]:
    c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=2, timeout_s=10.0)
    for b in [int(x) for x in os.environ.get("BS", "1,4,16,64,256,1024,4096,16384").split(",")]:
        send = synth.alltoall_sendbuf(b + p, p, b)
        want = oracle.alltoall_definition(send)
        for algo in ("pairwise", "bruck", "hier"):
            print("run", G, b, algo, flush=True)
            d_s = torch.from_numpy(send).cuda(); d_r = torch.zeros_like(d_s)
            c.alltoall(d_s, d_r, algo=algo)
            torch.cuda.synchronize()
            ok = np.array_equal(d_r.cpu().numpy(), want)
            if not ok: print("MISMATCH", G, b, algo, flush=True)
    c.finalize()
print("done")

"""Single-GPU alltoall p = P, SIZES_KIB: us per call under the CURRENT environment (knobs stay set)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm
from timing import t
p = int(os.environ.get("P", "32"))
c = Comm(ranks_per_proc=p, device=0)
row = {}
for b in [int(x) << 10 for x in os.environ.get("SIZES_KIB", "64").split(",")]:
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
    r = torch.empty_like(s)
    us = t(lambda: c.alltoall(s, r, algo="pairwise"), it=10)
    ok = bool(torch.equal(r.view(p, p, b).transpose(0, 1).reshape(p, p * b), s))
    row[b >> 10] = [round(us, 1), round(2 * p * p * b / us / 1e3 / 6543.7, 3), sorted(c.last_launch_path()), ok]
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MPXA_")}, "p": p, "KiB": row}), flush=True)

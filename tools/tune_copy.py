"""Time the hot workloads for one libmpxa build (MPXA_LIB selects a tuning variant)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm

def t(fn, it=20, w=3):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3

p = 8
c = Comm(ranks_per_proc=p, device=0)
res = {"lib": os.path.basename(os.environ.get("MPXA_LIB", "libmpxa.so")), "ns": os.environ.get("MPXA_NS"), "nf": os.environ.get("MPXA_NF")}
for b in (64 << 20, 4 << 20, 1 << 20):
    s = torch.randint(0, 255, (p, b), dtype=torch.uint8, device="cuda")
    r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
    us = t(lambda: c.allgather(s, r, algo="pairwise"))
    res[f"ag_{b>>20}M_us"] = round(us, 1); res[f"ag_{b>>20}M_hbm_tbs"] = round((p * b + p * p * b) / us / 1e6, 3)
    del s, r
for b in (16 << 20, 1 << 20):
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
    r = torch.empty_like(s)
    us = t(lambda: c.alltoall(s, r, algo="pairwise"))
    res[f"a2a_{b>>20}M_us"] = round(us, 1); res[f"a2a_{b>>20}M_hbm_tbs"] = round(2 * p * p * b / us / 1e6, 3)
    del s, r
if os.environ.get("COPY_REF"):
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda"); bb = torch.empty_like(a)
    us = t(lambda: bb.copy_(a)); res["torch_copy_1G_tbs"] = round(2 * (1 << 30) / us / 1e6, 3)
    a2 = torch.empty(4 << 30, dtype=torch.uint8, device="cuda"); s2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    us = t(lambda: a2.view(8, -1).copy_(s2.view(1, -1).expand(8, -1)))
    res["torch_bcast_512M_x8_tbs"] = round((4.5 * (1 << 30)) / us / 1e6, 3)
print(json.dumps(res), flush=True)

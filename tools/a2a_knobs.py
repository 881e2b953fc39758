"""Single-GPU alltoall at p = P ranks (env P, default 32), block sizes SIZES_KIB, under knob
settings KNOBS="A=1,B=2;C=3" ('' = defaults): device us per call (CUDA graph) and the
fraction of the measured HBM copy peak (read + write of every block)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2309_07337_b200 import Comm
from timing import t
p = int(os.environ.get("P", "32"))
peak = 6543.7
sizes = [int(x) << 10 for x in os.environ.get("SIZES_KIB", "64,256,1024").split(",")]
big = torch.randint(0, 255, (p * p * max(sizes),), dtype=torch.uint8, device="cuda")
for cfg in os.environ.get("KNOBS", "").split(";"):
    env = dict(kv.split("=") for kv in cfg.split(",") if kv)
    for k, v in env.items():
        os.environ[k] = v
    c = Comm(ranks_per_proc=p, device=0)
    for k in env:
        del os.environ[k]
    row = {}
    for b in sizes:
        s = big[: p * p * b].view(p, p * b)
        r = torch.empty_like(s)
        us = t(lambda: c.alltoall(s, r, algo="pairwise"), it=10)
        row[b >> 10] = [round(us, 1), round(2 * p * p * b / us / 1e3 / peak, 3), sorted(c.last_launch_path())]
        del r
    print(json.dumps({"knobs": cfg or "default", "p": p, "KiB: [us, frac, path]": row}), flush=True)
    c.finalize()

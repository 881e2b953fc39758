"""Single-GPU allgather p = 8, 2..64 MiB per rank: device us per call (CUDA graph) and the
fraction of the measured HBM copy peak, under dynamic-queue knob settings given as
KNOBS="NAME=V,NAME=V;NAME=V" (configurations separated by ';', '' = defaults)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2309_07337_b200 import Comm
from timing import t
p = 8
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6543.7
sizes = [int(x) << 20 for x in os.environ.get("SIZES_MIB", "2,4,8,16,64").split(",")]
big = torch.randint(0, 255, (p * max(sizes),), dtype=torch.uint8, device="cuda")
for cfg in os.environ.get("KNOBS", "").split(";"):
    env = dict(kv.split("=") for kv in cfg.split(",") if kv)
    for k, v in env.items():
        os.environ[k] = v
    c = Comm(ranks_per_proc=p, device=0)
    for k in env:
        del os.environ[k]
    row = {}
    for b in sizes:
        s = big[: p * b].view(p, b)
        r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
        us = t(lambda: c.allgather(s, r), it=5 if b >= (16 << 20) else 10)
        row[b >> 20] = [round(us, 1), round(9 * p * b / us / 1e3 / peak, 4)]
        del r
    print(json.dumps({"knobs": cfg or "default", "MiB: [us, frac]": row}), flush=True)
    c.finalize()

"""Small-message latency, single GPU p = P ranks (default 8; EMU = G emulated GPUs): alltoall and
allgather device us per call (CUDA graph of 200 calls) at SIZES bytes, under KNOBS="A=1;B=2"
('' = defaults), for the variants in ALGOS (default pairwise; allgather maps hier -> ring)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2309_07337_b200 import Comm
from timing import t
p = int(os.environ.get("P", "8"))
sizes = [int(x) for x in os.environ.get("SIZES", "16,256,4096").split(",")]
for cfg in os.environ.get("KNOBS", "").split(";"):
    env = dict(kv.split("=") for kv in cfg.split(",") if kv)
    for k, v in env.items():
        os.environ[k] = v
    c = Comm(ranks_per_proc=p, device=0, emulate_gpus=int(os.environ.get("EMU", "0")))
    for k in env:
        del os.environ[k]
    row = {}
    for algo in os.environ.get("ALGOS", "pairwise").split(","):
        sfx = "" if algo == "pairwise" else "_" + algo
        for b in sizes:
            s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
            r = torch.empty_like(s)
            row[f"a2a{sfx}_{b}"] = round(t(lambda: c.alltoall(s, r, algo=algo), it=200), 3)
            row[f"a2a{sfx}_{b}_path"] = sorted(c.last_launch_path())
            s2 = s[:, :b].contiguous()
            ag = "ring" if algo == "hier" else algo
            row[f"ag{sfx}_{b}"] = round(t(lambda: c.allgather(s2, r[:, : p * b], algo=ag), it=200), 3)
            row[f"ag{sfx}_{b}_path"] = sorted(c.last_launch_path())
    # the launch floor: a trivial torch copy of the same bytes
    x = torch.empty(16, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    row["torch_copy_16B"] = round(t(lambda: y.copy_(x), it=200), 3)
    print(json.dumps({"knobs": cfg or "default", "us": row}), flush=True)
    c.finalize()

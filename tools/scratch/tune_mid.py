"""Grid-shape sweep for mid/large messages on one GPU (p=8 ranks): TMA ring config
(MPXA_TMA_BIG) x column slices (MPXA_NS) x flow groups (MPXA_NF).  Env overrides are read
by mpxa_init, so every configuration gets a fresh communicator.  Prints JSON lines."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm

GS = torch.cuda.Stream()


def t(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=GS):
        for _ in range(it): fn()
    ts = []
    with torch.cuda.stream(GS):
        g.replay(); torch.cuda.synchronize()
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(GS); g.replay(); b.record(GS); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / it * 1e3)
    return sorted(ts)[1]


if __name__ == "__main__":
    p = 8
    sizes = [int(x) for x in os.environ.get("SIZES", str((256 << 10)) + "," + str(1 << 20) + "," + str(4 << 20) + "," + str(16 << 20)).split(",")]
    configs = [("auto", None, None, None)]
    for big in (0, 1):
        for ns in (148, 296, 592):
            if big and ns > 148 * 1: continue
            configs.append((f"big{big}_ns{ns}", big, ns, None))
        for nf in (2, 4, 8):
            configs.append((f"big{big}_nf{nf}", big, None, nf))
    big_buf = torch.randint(0, 255, (p * p * (16 << 20),), dtype=torch.uint8, device="cuda")
    out_buf = torch.empty_like(big_buf)
    for name, big, ns, nf in configs:
        for k, v in (("MPXA_TMA_BIG", big), ("MPXA_NS", ns), ("MPXA_NF", nf)):
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = str(v)
        c = Comm(ranks_per_proc=p, device=0)
        row = {"cfg": name}
        for b in sizes:
            s = big_buf[: p * p * b].view(p, p * b)
            r = out_buf[: p * p * b].view(p, p * b)
            us = t(lambda: c.alltoall(s, r, algo="pairwise", stream=GS))
            row[f"a2a_{b >> 10}K"] = [round(us, 1), round(2 * p * p * b / us / 1e6, 2)]
            s2 = big_buf[: p * b].view(p, b)
            us = t(lambda: c.allgather(s2, r, algo="pairwise", stream=GS))
            row[f"ag_{b >> 10}K"] = [round(us, 1), round((p * b + p * p * b) / us / 1e6, 2)]
        c.finalize()
        print(json.dumps(row), flush=True)

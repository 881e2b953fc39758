"""cfg4-shaped alltoallv timing on one GPU (p=8 ranks, int64, U{0..2 mean} counts, 10% zeros):
persistent request, device us per start/wait in a CUDA graph, HBM TB/s (read+write)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2309_07337_b200 import Comm
GS = torch.cuda.Stream()


def t(fn, it=20):
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


p = 8
c = Comm(ranks_per_proc=p, device=0)
res = {"nodyn": os.environ.get("MPXA_NO_DYN", "0")}
for mean in (64 << 10, 1 << 20, 4 << 20):
    for packed in (True, False):
        counts = synth.cfg4_counts(0, p, mean)
        sc = counts.astype(np.int64); rc = counts.T.copy()
        if packed:
            sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
            rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
        else:   # 8-byte gaps: half the segments 8 mod 16 apart
            sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc + 1, 1)[:, :-1]
            rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
        S = int((sd + sc).max()) * 8; R = int((rd + rc).max()) * 8
        s = torch.randint(0, 255, (p, S), dtype=torch.uint8, device="cuda")
        r = torch.zeros((p, R), dtype=torch.uint8, device="cuda")
        q = c.alltoallv_init(s, sc, sd, r, rc, rd, dtype_size=8)
        us = t(lambda: (q.start(GS), q.wait(GS)))
        moved = int(counts.sum()) * 8
        res[f"mean{mean >> 10}K_{'packed' if packed else 'gaps'}"] = [round(us, 1), round(2 * moved / us / 1e6, 2)]
        q.free()
print(json.dumps(res), flush=True)

"""Multi-step programs with uneven moves on one GPU: f1 locality-aware neighbor alltoallv
(sparse-matrix halo) and hierarchical alltoallv (cfg4 counts)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
p = 8
res = {"nodyn": os.environ.get("MPXA_NO_DYN", "0")}
gr, si, ri = synth.graph_from_edges(p, synth.spmv_edges(0, p, 1 << 20, 1 << 18, 3, contiguous=True))
ioff = np.concatenate([[0], np.cumsum(gr["indeg"])]); ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
srcs = [list(map(int, gr["src"][ioff[r]:ioff[r + 1]])) for r in range(p)]
dsts = [list(map(int, gr["dst"][ooff[r]:ooff[r + 1]])) for r in range(p)]
S = int((gr["sd"] + gr["sc"]).max()) * 8; Rb = int((gr["rd"] + gr["rc"]).max()) * 8
send_h, _ = synth.neighbor_buffers(1, p, gr, si, w=8)
c = Comm(ranks_per_proc=p, device=0, group_size=2)
topo = c.dist_graph_create_adjacent(srcs, dsts)
d_s = torch.from_numpy(send_h).cuda(); d_r = torch.zeros((p, Rb), dtype=torch.uint8, device="cuda")
q = c.neighbor_alltoallv_init(topo, d_s, gr["sc"], gr["sd"], d_r, gr["rc"], gr["rd"], dtype_size=8, send_indices=si, recv_indices=ri)
res["nb_locality_g2"] = round(t(lambda: (q.start(GS), q.wait(GS))), 1)
q.free()
for mean in (1 << 20, 4 << 20):
    counts = synth.cfg4_counts(0, p, mean)
    sc = counts.astype(np.int64); rc = counts.T.copy()
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
    s_ = torch.randint(0, 255, (p, int((sd + sc).max()) * 8), dtype=torch.uint8, device="cuda")
    r_ = torch.zeros((p, int((rd + rc).max()) * 8), dtype=torch.uint8, device="cuda")
    for algo in ("hier", "bruck"):
        q = c.alltoallv_init(s_, sc, sd, r_, rc, rd, dtype_size=8, algo=algo)
        res[f"a2av_{algo}_{mean >> 20}M"] = round(t(lambda: (q.start(GS), q.wait(GS))), 1)
        q.free()
print(json.dumps(res), flush=True)

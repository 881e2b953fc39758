"""A few launches of the locality-aware neighbor alltoallv over random sparse indices (the
small kernel's variable-piece mode), for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2309_07337_b200 import Comm
p, m, k = 8, 65536, 8192
gr, si, ri = synth.graph_from_edges(p, synth.spmv_edges(1, p, m, k, 3))
ioff = np.concatenate([[0], np.cumsum(gr["indeg"])]); ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
srcs = [list(map(int, gr["src"][ioff[r]:ioff[r + 1]])) for r in range(p)]
dsts = [list(map(int, gr["dst"][ooff[r]:ooff[r + 1]])) for r in range(p)]
send_h, r0 = synth.neighbor_buffers(1, p, gr, si, w=8)
c = Comm(ranks_per_proc=p, device=0, group_size=2)
topo = c.dist_graph_create_adjacent(srcs, dsts)
d_s, d_r = torch.from_numpy(send_h).cuda(), torch.from_numpy(r0).cuda()
q = c.neighbor_alltoallv_init(topo, d_s, gr["sc"], gr["sd"], d_r, gr["rc"], gr["rd"], dtype_size=8,
                              send_indices=si, recv_indices=ri)
for _ in range(5):
    q.start(); q.wait()
torch.cuda.synchronize()
print("ok")

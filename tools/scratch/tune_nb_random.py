"""f1 with a random sparse pattern (no runs): element-granular locality schedule."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth, oracle
from paper_2309_07337_b200 import Comm
import tune_mid
from tune_mid import t
tune_mid.GS = GS = torch.cuda.Stream()
p = 8
res = {}
chops = os.environ.get("CHOPS", "")   # "chop:tiles,..." -> MPXA_VAR_CHOP / MPXA_VAR_TILES
for m, k, chop in [(m, k, ch) for m, k in ((65536, 8192), (8192, 1024)) for ch in (chops.split(",") if chops else [""])]:
    if chop:
        a, _, b = chop.partition(":")
        os.environ["MPXA_VAR_CHOP"] = a
        if b: os.environ["MPXA_VAR_TILES"] = b
    gr, si, ri = synth.graph_from_edges(p, synth.spmv_edges(1, p, m, k, 3))
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])]); ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
    srcs = [list(map(int, gr["src"][ioff[r]:ioff[r + 1]])) for r in range(p)]
    dsts = [list(map(int, gr["dst"][ooff[r]:ooff[r + 1]])) for r in range(p)]
    send_h, r0 = synth.neighbor_buffers(1, p, gr, si, w=8)
    want = oracle.neighbor_definition(send_h, r0, 8, gr)
    c = Comm(ranks_per_proc=p, device=0, group_size=2)
    topo = c.dist_graph_create_adjacent(srcs, dsts)
    d_s = torch.from_numpy(send_h).cuda()
    for loc in (False, True):
        d_r = torch.from_numpy(r0).cuda()
        kw = dict(send_indices=si, recv_indices=ri) if loc else {}
        t0 = time.time()
        q = c.neighbor_alltoallv_init(topo, d_s, gr["sc"], gr["sd"], d_r, gr["rc"], gr["rd"], dtype_size=8, **kw)
        init_s = time.time() - t0
        q.start(GS); q.wait(GS); torch.cuda.synchronize()
        ok = bool(np.array_equal(d_r.cpu().numpy(), want))
        us = t(lambda: (q.start(GS), q.wait(GS)), it=5)
        res[f"m{m}_k{k}_{'loc' if loc else 'std'}{chop}"] = {"us": round(us, 1), "init_s": round(init_s, 2), "ok": ok}
        q.free()
    c.finalize()
print(json.dumps(res), flush=True)

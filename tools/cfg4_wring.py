"""cfg4 alltoallv (p = 8, mean 4 MiB) device time per persistent start+wait (CUDA graph):
int64 segments in warp-ring mode (default), with MPXA_NO_WRING=1 (LSU-register queue), int32
segments, and the same bytes as 16-B elements (all bulk TMA), also forced through the warp-ring mode."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import synth
from paper_2309_07337_b200 import Comm
import timing
from timing import t
GS = timing.GS
p = 8
res = {}
for name, elem, env in (("int64_wring", 8, {}), ("int64_wring_slack1", 8, {"MPXA_WSLACK": "1"}), ("int64_lsu", 8, {"MPXA_NO_WRING": "1"}), ("int32_wring", 4, {}),
                        ("16B_elements", 16, {}), ("16B_elements_wring", 16, {"MPXA_WRING": "2"})):
    for k, v in env.items():
        os.environ[k] = v
    c = Comm(ranks_per_proc=p, device=0)
    for k in env:
        del os.environ[k]
    for seed in (0, 1, 2):
        c4 = synth.cfg4_counts(seed, p, 4 << 20, elem=8)
        if elem != 8:
            c4 = c4 * 8 // elem
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed, c4, elem=elem)
        d_s = torch.from_numpy(send).cuda()
        d_r = torch.zeros((p, Rcap), dtype=torch.uint8, device="cuda")
        q = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, dtype_size=elem)
        us = t(lambda: (q.start(GS), q.wait(GS)), it=10)
        moved = int(sc.sum()) * elem
        res[f"{name}_seed{seed}"] = [round(us, 1), round(2 * moved / us / 1e6, 3), sorted(c.last_launch_path())]
        q.free()
        del d_s, d_r
    c.finalize()
print(json.dumps(res))

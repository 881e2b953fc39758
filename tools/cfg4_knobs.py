"""cfg4 alltoallv (p = 8) device time per persistent start+wait (CUDA graph) under knob sets
(VARIANTS='{"name": {"ENV": "val"}, ...}', first = reference), int64 and int32 segments
(ELEMS), means in MiB (MEANS), ODD=1 for counts that leave segments at every alignment; every
variant's output compared with the first's.  (Used for
the round-2 cp.async warp-ring experiment, MPXA_WLOAD, since removed: profiles/r02/shift_probe.txt.)"""
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
VARIANTS = tuple(json.loads(os.environ.get("VARIANTS", '{"default": {}}')).items())
comms = {}
for name, env in VARIANTS:
    for k, v in env.items():
        os.environ[k] = v
    comms[name] = Comm(ranks_per_proc=p, device=0)
    for k in env:
        del os.environ[k]
res = {}
for elem in (int(x) for x in os.environ.get("ELEMS", "8,4").split(",")):
    for mean in (float(x) for x in os.environ.get("MEANS", "1,2,4,8").split(",")):
        for seed in (0, 1):
            c4 = synth.cfg4_counts(seed, p, int(mean * (1 << 20)), elem=8) * 8 // elem
            if os.environ.get("ODD"):   # one more element per nonzero pair: offsets of every alignment
                c4 = c4 + (c4 > 0)
            send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed, c4, elem=elem)
            d_s = torch.from_numpy(send).cuda()
            ref = None
            for name, _ in VARIANTS:
                c = comms[name]
                d_r = torch.zeros((p, Rcap), dtype=torch.uint8, device="cuda")
                q = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, dtype_size=elem)
                us = t(lambda: (q.start(GS), q.wait(GS)), it=10)
                torch.cuda.synchronize()
                ok = True
                if ref is None:
                    ref = d_r.clone()
                else:
                    ok = bool(torch.equal(ref, d_r))
                moved = int(sc.sum()) * elem
                res[f"e{elem}_m{mean}_s{seed}_{name}"] = [round(us, 1), round(2 * moved / us / 1e3 / 6543.7, 4),
                                                         ok, sorted(c.last_launch_path())]
                q.free()
                del d_r
            del d_s, ref
print(json.dumps(res))

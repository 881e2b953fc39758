"""A/B of mid-size single-GPU alltoall / allgather (p = 8, device us per call in CUDA graphs)
between library builds: LIBS="name=path,name=path" (each run in a fresh process)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    from paper_2309_07337_b200 import Comm
    from timing import t
    p = 8
    c = Comm(ranks_per_proc=p, device=0)
    res = {}
    for b in [int(x) for x in os.environ.get("SIZES", "262144,1048576,2097152,4194304").split(",")]:
        s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
        r = torch.empty_like(s)
        res[f"a2a_{b}"] = round(t(lambda: c.alltoall(s, r, algo="pairwise"), it=20), 2)
        res[f"a2a_{b}_path"] = sorted(c.last_launch_path())
        s2 = s[:, :b].contiguous()
        res[f"ag_{b}"] = round(t(lambda: c.allgather(s2, r, algo="pairwise"), it=20), 2)
    print(json.dumps(res), flush=True)
else:
    for spec in os.environ.get("LIBS", "cur=paper_2309_07337_b200/libmpxa.so").split(","):
        name, path = spec.split("=")
        env = dict(os.environ, MPXA_LIB=os.path.join(ROOT, path))
        for rep in range(2):
            out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
            print(name, rep, out.stdout.strip() or out.stderr[-500:], flush=True)

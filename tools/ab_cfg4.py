"""A/B of cfg4 alltoallv (p = 8, int64, mean 4 MiB, persistent, CUDA graph) between library
builds: LIBS="name=path,..." (fresh process each, two repetitions)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import synth
    from paper_2309_07337_b200 import Comm
    from timing import t, GS
    p = 8
    c = Comm(ranks_per_proc=p, device=0)
    res = {}
    for seed in (0, 1, 2):
        c4 = synth.cfg4_counts(seed, p, 4 << 20)
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed, c4, elem=8)
        d_s = torch.from_numpy(send).cuda()
        d_r = torch.zeros((p, Rcap), dtype=torch.uint8, device="cuda")
        q = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, dtype_size=8, algo="pairwise")
        res[f"seed{seed}"] = round(t(lambda: (q.start(GS), q.wait(GS)), it=10), 1)
        q.free()
    print(json.dumps(res), flush=True)
else:
    for spec in os.environ.get("LIBS", "cur=paper_2309_07337_b200/libmpxa.so").split(","):
        name, path = spec.split("=")
        env = dict(os.environ, MPXA_LIB=os.path.join(ROOT, path))
        for rep in range(2):
            out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
            print(name, rep, out.stdout.strip() or out.stderr[-500:], flush=True)

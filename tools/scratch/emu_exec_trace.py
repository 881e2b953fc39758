"""Per-CTA start / end (globaltimer ns) of one emulated-GPU executor launch (MPXA_TRACE
build): p = 32 ranks on 8 emulated GPUs, pairwise alltoall at a few block sizes."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2309_07337_b200 import Comm, lib
L = lib()
p, G = int(os.environ.get("P", "32")), int(os.environ.get("EMU", "8"))
c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G)
for b in [int(x) for x in os.environ.get("SIZES", "16384,65536,262144").split(",")]:
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
    for _ in range(4): c.alltoall(s, r, algo="pairwise")
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 2048)()
    L.mpxa__cta_trace.argtypes = [ctypes.c_void_p]
    L.mpxa__cta_trace(None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.alltoall(s, r, algo="pairwise"); e1.record(); torch.cuda.synchronize()
    L.mpxa__cta_trace(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024).astype(np.int64)
    n = int((a[0] > 0).sum())
    st, en = a[0, :n], a[1, :n]
    t0 = st.min()
    q = lambda x: [int(np.percentile(x - t0, v)) for v in (0, 50, 90, 100)]
    print(b, "us", round(e0.elapsed_time(e1) * 1e3, 1), sorted(c.last_launch_path()), "ctas(row0)", n,
          "start", q(st), "end", q(en), flush=True)

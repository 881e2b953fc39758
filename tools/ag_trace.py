"""Per-CTA start / end (globaltimer) of single-GPU allgather launches, p = 8 ranks (MPXA_TRACE
build: MPXA_LIB=paper_2309_07337_b200/libmpxa_trace.so): where the fixed ~10 us per launch
above the HBM streaming time goes (ramp-up vs tail)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2309_07337_b200 import Comm, lib
L = lib()
p = 8
c = Comm(ranks_per_proc=p, device=0)
big = torch.randint(0, 255, (p * (64 << 20),), dtype=torch.uint8, device="cuda")
for b in [int(x) for x in os.environ.get("SIZES", str(4 << 20) + "," + str(16 << 20) + "," + str(64 << 20)).split(",")]:
    s = big[: p * b].view(p, b)
    r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
    for _ in range(4): c.allgather(s, r)
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 2048)()
    L.mpxa__cta_trace.argtypes = [ctypes.c_void_p]
    L.mpxa__cta_trace(None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.allgather(s, r); e1.record(); torch.cuda.synchronize()
    L.mpxa__cta_trace(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024).astype(np.int64)
    n = int((a[0] > 0).sum())
    st, en = a[0, :n], a[1, :n]
    t0 = st.min()
    q = lambda x: [round(float(np.percentile(x - t0, v)) / 1e3, 2) for v in (0, 10, 50, 90, 100)]
    ideal = 9 * p * b / 6543.7e9 * 1e6
    print(b >> 20, "MiB us", round(e0.elapsed_time(e1) * 1e3, 1), "ideal", round(ideal, 1), sorted(c.last_launch_path()),
          "ctas", n, "start_us", q(st), "end_us", q(en), flush=True)
    del r

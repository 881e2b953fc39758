"""Host cost per call of the one-shot alltoallv (cfg4 shape, p = 8 on one GPU): the Python
binding vs the bare C call with pre-marshalled pointers, vs persistent start/wait, and the
device time of the same launch.  One JSON line."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2309_07337_b200 import Comm
from paper_2309_07337_b200 import mpxa as M
p = 8
c = Comm(ranks_per_proc=p, device=0)
c4 = synth.cfg4_counts(0, p, 64)
send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c4, elem=8)
d_s = torch.from_numpy(send.view(np.int64)).cuda(); d_r = torch.zeros((p, Rcap // 8), dtype=torch.int64, device="cuda")
st = torch.cuda.Stream()
res = {}
N = 2000


def wall(fn):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N): fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / N * 1e6, 2)


res["python_one_shot_us"] = wall(lambda: c.alltoallv(d_s, sc, sd, d_r, rc, rd, dtype_size=8, stream=st))
L = M._lib()
arrs = [np.ascontiguousarray(a, np.int64) for a in (sc, sd, rc, rd)]
ptrs = [ctypes.c_void_p(a.ctypes.data) for a in arrs]
sp, rp = ctypes.c_void_p(d_s.data_ptr()), ctypes.c_void_p(d_r.data_ptr())
sb, rb = d_s.numel() * 8 // p, d_r.numel() * 8 // p
h, s_ = c.handle, ctypes.c_void_p(st.cuda_stream)
res["c_one_shot_us"] = wall(lambda: L.mpxa_alltoallv_algo(sp, ptrs[0], ptrs[1], sb, rp, ptrs[2], ptrs[3], rb, 8, 0, h, s_))
req = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, dtype_size=8)
res["python_persistent_us"] = wall(lambda: (req.start(st), req.wait(st)))
res["c_persistent_us"] = wall(lambda: (L.mpxa_start(req.handle, s_), L.mpxa_wait(req.handle, s_)))
print(json.dumps(res), flush=True)

# uniform one-shot alltoall (p = 8, 64 B blocks)
s8 = torch.randint(0, 255, (p, p * 64), dtype=torch.uint8, device="cuda"); r8 = torch.empty_like(s8)
res["python_alltoall_us"] = wall(lambda: c.alltoall(s8, r8, stream=st))
sp8, rp8 = ctypes.c_void_p(s8.data_ptr()), ctypes.c_void_p(r8.data_ptr())
res["c_alltoall_us"] = wall(lambda: L.mpxa_alltoall_algo(sp8, 64, 1, rp8, 0, h, s_))
print(json.dumps(res), flush=True)

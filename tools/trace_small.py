"""Phase stamps (%globaltimer, ns) of CTA 0 for small collectives (MPXA_TRACE build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_07337_b200 import Comm, lib
L = lib(); f = L.mpxa__trace; f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]; f.restype = ctypes.c_int
p = 8
c = Comm(ranks_per_proc=p, device=0)
for op, b in (("allgather", 4), ("alltoall", 4), ("allgather", 1024), ("alltoall", 1 << 20)):
    if op == "allgather":
        s = torch.zeros((p, b), dtype=torch.uint8, device="cuda"); r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
        fn = lambda: c.allgather(s, r, algo="pairwise")
    else:
        s = torch.zeros((p, p * b), dtype=torch.uint8, device="cuda"); r = torch.empty_like(s)
        fn = lambda: c.alltoall(s, r, algo="pairwise")
    for _ in range(5): fn()
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 32)()
    ctypes.memset(buf, 0, 256)
    f(c.handle, buf)
    t0 = buf[0]
    print(op, b, "producer:", [int(buf[i] - t0) if buf[i] else None for i in range(9)],
          "lsu warp1:", [int(buf[16 + i] - t0) if buf[16 + i] else None for i in range(9)], flush=True)
    for i in range(32): buf[i] = 0

"""A few launches of one collective at one size (for ncu captures of one kernel path).
OP=alltoall|allgather|alltoallv, ALGO, B (block bytes; alltoallv: cfg4 mean), EMU (emulated
GPUs), P (ranks, default 8), N (launches, default 5); knobs through the MPXA_* environment."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2309_07337_b200 import Comm
p = int(os.environ.get("P", "8"))
b = int(os.environ.get("B", "16"))
op = os.environ.get("OP", "alltoall")
algo = os.environ.get("ALGO", "pairwise")
n = int(os.environ.get("N", "5"))
c = Comm(ranks_per_proc=p, device=0, emulate_gpus=int(os.environ.get("EMU", "0")), group_size=2)
if op == "alltoallv":
    counts = synth.cfg4_counts(0, p, b)
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, counts, elem=8)
    s = torch.from_numpy(send).cuda()
    r = torch.zeros((p, Rcap), dtype=torch.uint8, device="cuda")
    q = c.alltoallv_init(s, sc, sd, r, rc, rd, dtype_size=8, algo=algo)
    fn = lambda: (q.start(), q.wait())
elif op == "allgather":
    s = torch.randint(0, 255, (p, b), dtype=torch.uint8, device="cuda")
    r = torch.empty((p, p * b), dtype=torch.uint8, device="cuda")
    fn = lambda: c.allgather(s, r, algo=algo)
else:
    s = torch.randint(0, 255, (p, p * b), dtype=torch.uint8, device="cuda")
    r = torch.empty_like(s)
    fn = lambda: c.alltoall(s, r, algo=algo)
for _ in range(n):
    fn()
torch.cuda.synchronize()
assert c.check() == 0
print("ok", sorted(c.last_launch_path()))

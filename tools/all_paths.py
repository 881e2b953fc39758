"""A compact run over every kernel path (compute-sanitizer is closed on this pool, so this is
a plain run, each result checked against the oracle): the tiny kernels (one-step, multi-step one CTA and owned flows, eager),
the small kernel (8-B path), the exec kernel (static, dynamic single-step, dynamic multi-step,
warp rings), the emulated multi-GPU protocol, alltoallv (misaligned), neighbor (standard /
locality), partitioned.  The oracle is test infrastructure: this is a test driver.
PARTS=tiny,core,wring,nb,part selects a subset (default: all)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle, synth
from paper_2309_07337_b200 import Comm

dev = "cuda"
ok = True
PARTS = os.environ.get("PARTS", "tiny,core,wring,nb,part").split(",")


def check(name, got, want):
    global ok
    good = np.array_equal(got, want)
    ok &= good
    if not good:
        print("MISMATCH", name, flush=True)


if "tiny" in PARTS:
    p = 8
    for G in (0, 4):
        c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=2, timeout_s=60.0)
        for b in (16, 24, 4096 + 8):
            send = synth.alltoall_sendbuf(b, p, b)
            for algo in ("pairwise", "bruck", "hier"):
                d = torch.from_numpy(send).to(dev); r = torch.zeros_like(d)
                c.alltoall(d, r, algo=algo); torch.cuda.synchronize()
                check(("tiny a2a", G, b, algo, sorted(c.last_launch_path())), r.cpu().numpy(), oracle.alltoall_definition(send))
            ag = send[:, :b].copy()
            for algo in ("pairwise", "bruck", "ring"):
                r = torch.zeros((p, p * b), dtype=torch.uint8, device=dev)
                c.allgather(torch.from_numpy(ag).to(dev), r, algo=algo); torch.cuda.synchronize()
                check(("tiny ag", G, b, algo, sorted(c.last_launch_path())), r.cpu().numpy(), oracle.allgather_definition(ag))
        cnt = synth.cfg4_counts(3, p, 64)
        send, sc, sd, rc, rd, S, Rc = synth.alltoallv_buffers(3, cnt, elem=8, packed=False)
        r0 = np.full((p, Rc), 0xA5, np.uint8)
        r = torch.from_numpy(r0).to(dev)
        c.alltoallv(torch.from_numpy(send).to(dev), sc, sd, r, rc, rd, algo="pairwise", dtype_size=8)
        torch.cuda.synchronize()
        check(("small a8", G), r.cpu().numpy(), oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, r0))
        c.finalize()

if "wring" in PARTS:
    os.environ["MPXA_WRING"] = "2"          # the warp rings at a size the sanitizer finishes
    p = 8
    c = Comm(ranks_per_proc=p, device=0, timeout_s=120.0)
    del os.environ["MPXA_WRING"]
    for elem in (8, 4, 1):
        cnt = synth.cfg4_counts(5, p, 96 << 10, elem=8) * 8 // elem
        send, sc, sd, rc, rd, S, Rc = synth.alltoallv_buffers(5, cnt, elem=elem, packed=False)
        r0 = np.full((p, Rc), 0xA5, np.uint8)
        r = torch.from_numpy(r0).to(dev)
        c.alltoallv(torch.from_numpy(send).to(dev), sc, sd, r, rc, rd, algo="pairwise", dtype_size=elem)
        torch.cuda.synchronize()
        check(("wring", elem, sorted(c.last_launch_path())), r.cpu().numpy(),
              oracle.alltoallv_definition(send, sc, sd, rc, rd, elem, r0))
    ag = np.random.default_rng(7).integers(0, 256, (p, (1 << 20) + 24), dtype=np.uint8)
    r = torch.zeros((p, p * ag.shape[1]), dtype=torch.uint8, device=dev)
    c.allgather(torch.from_numpy(ag).to(dev), r, algo="pairwise"); torch.cuda.synchronize()
    check(("wring ag", sorted(c.last_launch_path())), r.cpu().numpy(), oracle.allgather_definition(ag))
    c.finalize()

for p, G in (((4, 0), (8, 0), (8, 2)) if "core" in PARTS else ()):
    c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, timeout_s=60.0)
    for b in (4, 1000, 65536, 1 << 20):
        send = np.random.default_rng(b).integers(0, 256, (p, p * b), dtype=np.uint8)
        want = oracle.alltoall_definition(send)
        for algo in ("pairwise", "bruck", "hier"):
            d = torch.from_numpy(send).to(dev); r = torch.zeros_like(d)
            c.alltoall(d, r, algo=algo); torch.cuda.synchronize()
            check(("a2a", p, G, b, algo), r.cpu().numpy(), want)
        ag = send[:, :b].copy(); agw = oracle.allgather_definition(ag)
        for algo in ("pairwise", "bruck", "ring", "hier"):
            r = torch.zeros((p, p * b), dtype=torch.uint8, device=dev)
            c.allgather(torch.from_numpy(ag).to(dev), r, algo=algo); torch.cuda.synchronize()
            check(("ag", p, G, b, algo), r.cpu().numpy(), agw)
    cnt = synth.cfg4_counts(1, p, 300000)
    send, sc, sd, rc, rd, S, Rc = synth.alltoallv_buffers(1, cnt, elem=8, packed=False)
    r0 = np.full((p, Rc), 0xA5, np.uint8)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, r0)
    for algo in ("pairwise", "hier", "bruck"):
        r = torch.from_numpy(r0).to(dev)
        c.alltoallv(torch.from_numpy(send).to(dev), sc, sd, r, rc, rd, algo=algo, dtype_size=8)
        torch.cuda.synchronize()
        check(("a2av", p, G, algo), r.cpu().numpy(), want)
    c.finalize()
if "nb" in PARTS:
    p = 8
    gr, si, ri = synth.graph_from_edges(p, synth.spmv_edges(2, p, 4096, 1024, 3, contiguous=True))
    send, r0 = synth.neighbor_buffers(0, p, gr, si)
    want = oracle.neighbor_definition(send, r0, 8, gr)
    c = Comm(ranks_per_proc=p, device=0, group_size=2)
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])]); ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
    topo = c.dist_graph_create_adjacent([list(map(int, gr["src"][ioff[r]:ioff[r + 1]])) for r in range(p)],
                                        [list(map(int, gr["dst"][ooff[r]:ooff[r + 1]])) for r in range(p)])
    for kw in ({}, dict(send_indices=si, recv_indices=ri)):
        r = torch.from_numpy(r0).to(dev)
        q = c.neighbor_alltoallv_init(topo, torch.from_numpy(send).to(dev), gr["sc"], gr["sd"], r, gr["rc"], gr["rd"],
                                      dtype_size=8, **kw)
        q.start(); q.wait(); torch.cuda.synchronize()
        check(("neighbor", bool(kw)), r.cpu().numpy(), want)
        q.free()
if "part" in PARTS:
    s = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device=dev); rb = torch.zeros_like(s)
    c2 = Comm(ranks_per_proc=2, device=0)
    ps = c2.psend_init(s, 4, 0, 1); pr = c2.precv_init(rb, 2, 1, 0); c2.pmatch()
    pr.start(); ps.start(); ps.pready(0, 4); ps.wait(); pr.wait(); torch.cuda.synchronize()
    check("partitioned", s.cpu().numpy(), rb.cpu().numpy())
print("sanitize case ok" if ok else "MISMATCH")
sys.exit(0 if ok else 1)

"""Multi-process setup on ONE GPU (-m gpu): two processes, gloo bootstrap, CUDA IPC.

Only the collective SETUP path runs here (mpxa_init's bootstrap all-gather and IPC
exchange of the symmetric regions and workspace, mpxa_register's window exchange, argument
checks that fail before any kernel launches).  No collective kernel is launched: kernels
that wait on each other must not run as separate launches on one GPU (B200_PROFILING.md),
so the device protocol itself is covered by the emulated multi-GPU tests.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WS = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _body(rank, port, q):
    import sys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=WS)
        torch.cuda.set_device(0)
        from paper_2309_07337_b200 import Comm, MpxaError
        from paper_2309_07337_b200 import mpxa as M
        c = Comm(ranks_per_proc=2, device=0, pg=dist.group.WORLD, heap_bytes=8 << 20)
        assert c.p == 4 and c.nprocs == 2 and c.proc == rank
        send = torch.zeros(2 * 4 * 64, dtype=torch.uint8, device="cuda")
        recv = torch.zeros_like(send)
        # unregistered recvbuf: rejected before any data moves, identically on both processes
        try:
            c.alltoall(send, recv)
            raise AssertionError("expected MPXA_ERR_UNREGISTERED")
        except MpxaError as e:
            assert e.status == M.ERR_UNREGISTERED
        c.register(recv)
        c.register(recv)           # already registered everywhere: no new window
        # f1: topology all-gather + persistent neighbor init (standard / locality-aware): the
        # global graph is assembled from both processes' rank lists and compiled once
        r0 = 2 * rank
        srcs = [[(r0 + t - 1) % 4, (r0 + t + 1) % 4] for t in range(2)]
        topo = c.dist_graph_create_adjacent(srcs, srcs)
        nb_s = torch.zeros(2 * 2 * 8, dtype=torch.int64, device="cuda")
        nb_r = torch.zeros(2 * 2 * 8, dtype=torch.int64, device="cuda")
        sc = [8, 8, 8, 8]
        sd = [0, 8, 0, 8]
        ids = []
        for t in range(2):
            for d in ((r0 + t - 1) % 4, (r0 + t + 1) % 4):
                ids += [(r0 + t) * 1000 + d * 10 + k for k in range(8)]
        rids = []
        for t in range(2):
            for src in ((r0 + t - 1) % 4, (r0 + t + 1) % 4):
                rids += [src * 1000 + (r0 + t) * 10 + k for k in range(8)]
        for kw in ({}, dict(send_indices=ids, recv_indices=rids)):
            req = c.neighbor_alltoallv_init(topo, nb_s, sc, sd, nb_r, sc, sd, **kw)
            req.free()
        topo.free()
        # f3: partitioned channels across the two processes -- the single match maps the
        # peer's receive buffer and flag heap (no kernels: they would wait on each other)
        ps_buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
        pr_buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
        ps = c.psend_init(ps_buf, 4, r0, (r0 + 2) % 4, 7)
        pr = c.precv_init(pr_buf, 2, r0, (r0 + 2) % 4, 7)
        c.pmatch()
        assert len(ps.device_handle()) == 128
        ps.free(); pr.free()
        lonely = c.psend_init(ps_buf, 4, r0, (r0 + 2) % 4, 99) if rank == 0 else None
        try:
            c.pmatch()
            raise AssertionError("expected MPXA_ERR_MISMATCH")
        except MpxaError as e:
            assert e.status == M.ERR_MISMATCH
        if lonely is not None:
            lonely.free()
        assert c.launch_count() == 0
        c.finalize()
        # topology mismatch across processes
        try:
            Comm(ranks_per_proc=2 + rank, device=0, pg=dist.group.WORLD, heap_bytes=1 << 20)
            raise AssertionError("expected MPXA_ERR_MISMATCH")
        except MpxaError as e:
            assert e.status == M.ERR_MISMATCH
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))


def test_two_process_init_ipc_register():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_body, args=(r, port, q)) for r in range(WS)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r, msg in res:
        assert msg == "ok", f"rank {r}: {msg}"

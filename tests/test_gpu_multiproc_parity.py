"""Multi-process parity: one process per visible GPU, the real IPC / NVLink path (-m gpu).

Skipped below 2 visible GPUs (one process per GPU; ranks whose kernels wait on one another
must never share a GPU -- B200_PROFILING.md).  Every process hosts R ranks of the
communicator; its buffers hold its R rows of the global seeded inputs (synth/), and its
received rows are compared bit-exactly with the oracle's definitions (oracle/):

  * alltoall pairwise / Bruck / hierarchical and allgather direct / Bruck / ring /
    hierarchical at sizes in the eager range (<= 128 KiB per GPU pair), the direct
    (clear-to-send + flags) range and the dynamic work-queue range, R = 1 and 2;
  * alltoallv pairwise / hierarchical / Bruck-v (cfg4 counts, gapped displacements, 0xA5
    canaries outside the received ranges) and the device counts exchange + scan;
  * persistent requests: 100 start/wait cycles, on recv buffers NOT registered by the caller
    (the *_init binds them), fresh data checked at cycles 0, 1 and 99;
  * a partitioned channel between ranks on different GPUs;
  * a deliberately ragged call order (one process calls a collective the others skip) that
    must end in MPXA_ERR_TIMEOUT from the device watchdog, not a hang.

PAPER.md:113-114 (MPIX_Comm_init), PAPER.md:168 (GPU data path); SURVEY.md §8(e)."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import mp_util  # noqa: E402

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
need2 = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (one process per GPU)")


def _setup(rank):
    sys.path.insert(0, ROOT)
    torch.cuda.set_device(rank)
    return f"cuda:{rank}"


def _collectives(rank, world, R):
    import torch.distributed as dist
    import oracle
    import synth
    from paper_2309_07337_b200 import Comm
    dev = _setup(rank)
    p = world * R
    rows = slice(rank * R, (rank + 1) * R)
    c = Comm(ranks_per_proc=R, device=rank, pg=dist.group.WORLD, group_size=R, timeout_s=30.0)
    cg = Comm(ranks_per_proc=R, device=rank, pg=dist.group.WORLD, group_size=max(1, (p // 2)), timeout_s=30.0) \
        if p >= 4 else None
    # (host memory: every process builds the global p x p*b input and the oracle's result)
    for b in (16, 1000, 300_000, (4 << 20) if p <= 8 else (1 << 20)):
        send_all = synth.alltoall_sendbuf(b % 97, p, b)
        want = oracle.alltoall_definition(send_all)
        d_s = torch.from_numpy(send_all[rows].copy()).to(dev)
        d_r = torch.empty_like(d_s)
        c.register(d_r)                 # (windows are per comm: register with each)
        if cg:
            cg.register(d_r)
        for cc, algo in ((c, "pairwise"), (c, "bruck"), (c, "hier")) + (((cg, "hier"),) if cg else ()):
            d_r.fill_(0xA5)
            torch.cuda.synchronize()
            dist.barrier()
            cc.alltoall(d_s, d_r, algo=algo)
            torch.cuda.synchronize()
            assert cc.check() == 0, (b, algo)
            assert np.array_equal(d_r.cpu().numpy(), want[rows]), ("alltoall", b, algo)
        ag = synth.allgather_sendbuf(b % 89, p, b)
        agw = oracle.allgather_definition(ag)
        g_s = torch.from_numpy(ag[rows].copy()).to(dev)
        g_r = torch.empty((R, p * b), dtype=torch.uint8, device=dev)
        c.register(g_r)
        for algo in ("pairwise", "bruck", "ring", "hier"):
            g_r.fill_(0x5A)
            torch.cuda.synchronize()
            dist.barrier()
            c.allgather(g_s, g_r, algo=algo)
            torch.cuda.synchronize()
            assert c.check() == 0, (b, algo)
            assert np.array_equal(g_r.cpu().numpy(), agw[rows]), ("allgather", b, algo)
        del d_s, d_r, g_s, g_r
    # alltoallv (cfg4 counts, gapped displacements, canaries) -- three means
    for mean in (64, 64 << 10, (1 << 20) if p <= 8 else (256 << 10)):
        counts = synth.cfg4_counts(1, p, mean)
        send_all, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(1, counts, elem=8, packed=False)
        recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
        want = oracle.alltoallv_definition(send_all, sc, sd, rc, rd, 8, recv0)
        d_s = torch.from_numpy(send_all[rows].copy()).to(dev)
        d_r = torch.from_numpy(recv0[rows].copy()).to(dev)
        c.register(d_r)
        if cg:
            cg.register(d_r)
        for cc, algo in ((c, "pairwise"), (c, "hier"), (c, "bruck")) + (((cg, "hier"),) if cg else ()):
            d_r.copy_(torch.from_numpy(recv0[rows].copy()).to(dev))
            torch.cuda.synchronize()
            dist.barrier()
            cc.alltoallv(d_s, sc[rows].copy(), sd[rows].copy(), d_r, rc[rows].copy(), rd[rows].copy(), algo=algo,
                         dtype_size=8)
            torch.cuda.synchronize()
            assert cc.check() == 0, (mean, algo)
            assert np.array_equal(d_r.cpu().numpy(), want[rows]), ("alltoallv", mean, algo)
        # device counts exchange + scan (A2): recvcounts = transpose, rdispls = exclusive scan
        d_sc = torch.from_numpy(sc[rows].copy()).to(dev)
        d_rc = torch.zeros_like(d_sc)
        d_rd = torch.zeros_like(d_sc)
        dist.barrier()
        c.alltoallv_counts(d_sc, d_rc, d_rd)
        torch.cuda.synchronize()
        rc_w, rd_w, _ = oracle.counts_exchange(sc)
        assert np.array_equal(d_rc.cpu().numpy(), rc_w[rows]) and np.array_equal(d_rd.cpu().numpy(), rd_w[rows])
    if cg:
        cg.finalize()
    c.finalize()


def _persistent(rank, world, R):
    import torch.distributed as dist
    import oracle
    import synth
    from paper_2309_07337_b200 import Comm
    dev = _setup(rank)
    p = world * R
    rows = slice(rank * R, (rank + 1) * R)
    c = Comm(ranks_per_proc=R, device=rank, pg=dist.group.WORLD, timeout_s=30.0)
    for b, algo in ((64, "pairwise"), (2000, "bruck"), (1 << 20, "pairwise")):
        d_s = torch.empty((R, p * b), dtype=torch.uint8, device=dev)
        d_r = torch.empty_like(d_s)                   # not registered by the caller
        req = c.alltoall_init(d_s, d_r, algo=algo)
        for cyc in range(100):
            if cyc in (0, 1, 99):
                send_all = synth.alltoall_sendbuf(1000 * b + cyc, p, b)
                d_s.copy_(torch.from_numpy(send_all[rows].copy()).to(dev))
                d_r.zero_()
                torch.cuda.synchronize()
                dist.barrier()
            req.start()
            req.wait()
            if cyc in (0, 1, 99):
                torch.cuda.synchronize()
                assert np.array_equal(d_r.cpu().numpy(), oracle.alltoall_definition(send_all)[rows]), (b, cyc)
        req.free()
    # persistent alltoallv, cfg4 64 KiB mean
    counts = synth.cfg4_counts(2, p, 64 << 10)
    send_all, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(2, counts, elem=8, packed=True)
    recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send_all, sc, sd, rc, rd, 8, recv0)
    d_s = torch.from_numpy(send_all[rows].copy()).to(dev)
    d_r = torch.from_numpy(recv0[rows].copy()).to(dev)
    req = c.alltoallv_init(d_s, sc[rows].copy(), sd[rows].copy(), d_r, rc[rows].copy(), rd[rows].copy(),
                           dtype_size=8)
    torch.cuda.synchronize()
    dist.barrier()
    for cyc in range(100):
        req.start()
        req.wait()
    torch.cuda.synchronize()
    assert np.array_equal(d_r.cpu().numpy(), want[rows])
    req.free()
    assert c.check() == 0
    c.finalize()


def _partitioned(rank, world, R):
    import torch.distributed as dist
    from paper_2309_07337_b200 import Comm
    dev = _setup(rank)
    c = Comm(ranks_per_proc=R, device=rank, pg=dist.group.WORLD, timeout_s=30.0)
    nbytes = 8 << 20
    src, dst = 0, R * (world - 1)                     # first rank of GPU 0 -> first rank of the last GPU
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    buf = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev, generator=gen)
    req = None
    if rank == 0:
        req = c.psend_init(buf, 8, src, dst)
    elif rank == world - 1:
        buf.zero_()
        req = c.precv_init(buf, 4, dst, src)
    c.pmatch()
    for cyc in range(3):
        torch.cuda.synchronize()
        dist.barrier()
        if req is not None:
            req.start()
            if rank == 0:
                req.pready(0, 8)
            req.wait()
        torch.cuda.synchronize()
    if rank == world - 1:
        gen.manual_seed(5)
        want = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev, generator=gen)
        assert torch.equal(buf, want)
    dist.barrier()
    if req is not None:
        req.free()
    assert c.check() == 0
    c.finalize()


def _ragged(rank, world, R):
    import torch.distributed as dist
    from paper_2309_07337_b200 import Comm
    from paper_2309_07337_b200 import mpxa as M
    _setup(rank)
    p = world * R
    for b in (64, 1 << 20):                           # eager and direct protocols, fresh comm each
        c = Comm(ranks_per_proc=R, device=rank, pg=dist.group.WORLD, timeout_s=2.0)
        d_s = torch.zeros((R, p * b), dtype=torch.uint8, device=f"cuda:{rank}")
        d_r = torch.zeros_like(d_s)
        c.register(d_r)
        if rank == 0:                                 # the others never make this call
            c.alltoall(d_s, d_r, algo="pairwise")
            torch.cuda.synchronize()
            assert c.check() == M.ERR_TIMEOUT, b
        dist.barrier()
        c.finalize()


@need2
@pytest.mark.parametrize("R", [1, 2])
def test_collectives_all_variants(R):
    mp_util.spawn(_collectives, NGPU, R, timeout=900)


@need2
@pytest.mark.parametrize("R", [1, 2])
def test_persistent_100_cycles_unregistered_recv(R):
    mp_util.spawn(_persistent, NGPU, R, timeout=900)


@need2
def test_partitioned_across_gpus():
    mp_util.spawn(_partitioned, NGPU, 2)


@need2
def test_ragged_call_order_times_out():
    mp_util.spawn(_ragged, NGPU, 1, timeout=300)

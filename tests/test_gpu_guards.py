"""Guard bands around every receive buffer (-m gpu): no launch path writes outside the buffer
it was given.

compute-sanitizer is closed on this pool, so out-of-bounds writes are caught the direct way:
each recv buffer is a view into a larger allocation whose bytes before and after it are
filled with 0x5A; after the collective the view must equal the oracle's result (oracle/)
AND every guard byte must still be 0x5A.  The views start at offsets 0, 8 and 1 from a 16-B
boundary, so the aligned, 8-byte and byte-granular paths all run, over every launch path:
tiny kernels, the small kernel, the eager protocol (emulated GPUs), the static executor, the
dynamic work queues and the warp rings (MPXA_WRING=2).  SURVEY.md §8(b): the library
writes only [recvbuf, recvbuf + R * recv_bytes)."""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2309_07337_b200 import Comm  # noqa: E402

DEV = "cuda:0"
GUARD = 4096
_COMMS = {}


def comm(p, G=0, g=0, wring=False):
    key = (p, G, g, wring)
    if key not in _COMMS:
        if wring:
            os.environ["MPXA_WRING"] = "2"
        try:
            _COMMS[key] = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=g, timeout_s=20.0)
        finally:
            os.environ.pop("MPXA_WRING", None)
    return _COMMS[key]


def guarded(rows, cols, off):
    """(backing, view): view = rows x cols bytes at byte offset GUARD + off of a 0x5A backing."""
    back = torch.full((2 * GUARD + off + rows * cols,), 0x5A, dtype=torch.uint8, device=DEV)
    return back, back[GUARD + off: GUARD + off + rows * cols].view(rows, cols)


def check_guards(back, off, n):
    b = back.cpu().numpy()
    lo, hi = b[: GUARD + off], b[GUARD + off + n:]
    assert (lo == 0x5A).all(), ("below", int(np.flatnonzero(lo != 0x5A)[-1]) - (GUARD + off))
    assert (hi == 0x5A).all(), ("above", int(np.flatnonzero(hi != 0x5A)[0]))


@pytest.mark.parametrize("off", [0, 8, 1])
@pytest.mark.parametrize("G", [0, 2, 4])
def test_alltoall_guards(off, G):
    p = 8
    c = comm(p, G, 2)
    sizes = (16, 1000, 4096 + 12, 65536 + 128) + ((2 << 20) + 8,) * (G == 0)
    for b in sizes:
        send = synth.alltoall_sendbuf(b + off, p, b)
        want = oracle.alltoall_definition(send)
        d_s = torch.from_numpy(send).to(DEV)
        for algo in ("pairwise", "bruck", "hier"):
            back, recv = guarded(p, p * b, off)
            c.alltoall(d_s, recv, algo=algo)
            torch.cuda.synchronize()
            assert c.check() == 0
            assert np.array_equal(recv.cpu().numpy(), want), (b, algo, sorted(c.last_launch_path()))
            check_guards(back, off, p * p * b)


@pytest.mark.parametrize("off", [0, 8, 1])
@pytest.mark.parametrize("G", [0, 2, 4])
def test_allgather_guards(off, G):
    p = 8
    c = comm(p, G, 2)
    sizes = (16, 1000, 4096 + 12, 300_000) + ((8 << 20) + 8,) * (G == 0)
    for b in sizes:
        ag = synth.allgather_sendbuf(b + off, p, b)
        want = oracle.allgather_definition(ag)
        d_s = torch.from_numpy(ag).to(DEV)
        for algo in ("pairwise", "bruck", "ring", "hier"):
            back, recv = guarded(p, p * b, off)
            c.allgather(d_s, recv, algo=algo)
            torch.cuda.synchronize()
            assert c.check() == 0
            assert np.array_equal(recv.cpu().numpy(), want), (b, algo, sorted(c.last_launch_path()))
            check_guards(back, off, p * p * b)


@pytest.mark.parametrize("off", [0, 8])
@pytest.mark.parametrize("G,wring", [(0, False), (0, True), (2, False)])
def test_alltoallv_guards(off, G, wring):
    """cfg4 counts (int64, gapped displacements, 0xA5 outside the received ranges) at means
    64 B / 64 KiB / 1 MiB; the recv row capacity ends exactly at the last received byte of
    the fullest row, so a tail overrun reaches the guard."""
    p = 8
    c = comm(p, G, 2, wring)
    for mean in (64, 64 << 10, 1 << 20):
        counts = synth.cfg4_counts(off + 7, p, mean)
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(off + 7, counts, elem=8, packed=False)
        recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
        want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0)
        d_s = torch.from_numpy(send).to(DEV)
        for algo in ("pairwise", "hier", "bruck"):
            back, recv = guarded(p, Rcap, off)
            recv.copy_(torch.from_numpy(recv0).to(DEV))
            c.alltoallv(d_s, sc, sd, recv, rc, rd, algo=algo, dtype_size=8)
            torch.cuda.synchronize()
            assert c.check() == 0
            assert np.array_equal(recv.cpu().numpy(), want), (mean, algo, sorted(c.last_launch_path()))
            check_guards(back, off, p * Rcap)


@pytest.mark.parametrize("off", [0, 8])
@pytest.mark.parametrize("loc", [False, True])
def test_neighbor_guards(off, loc):
    """Persistent neighborhood alltoallv (standard and locality-aware dedup), halo-exchange
    topology, 3 start/wait cycles."""
    p = 8
    gr, si, ri = synth.graph_from_edges(p, synth.spmv_edges(2, p, 4096, 1024, 3, contiguous=True))
    send, r0 = synth.neighbor_buffers(0, p, gr, si)
    want = oracle.neighbor_definition(send, r0, 8, gr)
    c = Comm(ranks_per_proc=p, device=0, group_size=2, timeout_s=20.0)
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])])
    ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
    topo = c.dist_graph_create_adjacent([list(map(int, gr["src"][ioff[r]:ioff[r + 1]])) for r in range(p)],
                                        [list(map(int, gr["dst"][ooff[r]:ooff[r + 1]])) for r in range(p)])
    kw = dict(send_indices=si, recv_indices=ri) if loc else {}
    back, recv = guarded(p, r0.shape[1], off)
    recv.copy_(torch.from_numpy(r0).to(DEV))
    q = c.neighbor_alltoallv_init(topo, torch.from_numpy(send).to(DEV), gr["sc"], gr["sd"], recv, gr["rc"],
                                  gr["rd"], dtype_size=8, **kw)
    for _ in range(3):
        q.start()
        q.wait()
    torch.cuda.synchronize()
    assert np.array_equal(recv.cpu().numpy(), want)
    check_guards(back, off, p * r0.shape[1])
    q.free()
    assert c.check() == 0
    c.finalize()


@pytest.mark.parametrize("off", [0, 8, 1])
@pytest.mark.parametrize("nbytes,ps,pr", [(1000, 4, 2), (1 << 20, 16, 4), ((4 << 20) + 32, 4, 16)])
def test_partitioned_guards(off, nbytes, ps, pr):
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=DEV)
    back, rb = guarded(1, nbytes, off)
    rb = rb.view(-1)
    s = c.psend_init(src, ps, 0, 1)
    r = c.precv_init(rb, pr, 1, 0)
    c.pmatch()
    r.start()
    s.start()
    s.pready(0, ps)
    s.wait()
    r.wait()
    torch.cuda.synchronize()
    assert torch.equal(src, rb)
    check_guards(back, off, nbytes)
    s.free()
    r.free()
    assert c.check() == 0
    c.finalize()

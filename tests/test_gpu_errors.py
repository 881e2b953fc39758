"""The boundary's error contract (SURVEY.md §8(b) "Errors"; -m gpu).

Every argument error of the core collectives and their persistent *_init forms is detected
BEFORE any data moves ("argument error before any send"): the call returns the
documented status, no kernel is launched (launch counter unchanged) and the receive buffer's
0xA5 canary is untouched.  Codes: MPXA_ERR_ARG (NULL, overlap, negative count, displacement +
count beyond capacity, dtype_size not in {1,2,4,8,16}), MPXA_ERR_MISMATCH (sendcounts^T !=
recvcounts), MPXA_ERR_TOPOLOGY (p % g != 0), MPXA_ERR_ALGO (a
variant the op does not have), MPXA_ERR_LIFECYCLE."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2309_07337_b200 import Comm, MpxaError  # noqa: E402
from paper_2309_07337_b200 import mpxa as M  # noqa: E402

DEV = "cuda:0"
P = 4


@pytest.fixture(scope="module")
def c():
    cm = Comm(ranks_per_proc=P, device=0, group_size=2, timeout_s=20.0)
    yield cm
    cm.finalize()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _expect(c, status, fn, canary):
    """fn() must fail with `status`, launch nothing and leave the canary intact."""
    n0 = c.launch_count()
    rc = fn()
    assert rc == status, (rc, status)
    torch.cuda.synchronize()
    assert c.launch_count() == n0
    assert bool((canary == 0xA5).all())


def _bufs(b):
    s = torch.randint(0, 256, (P, P * b), dtype=torch.uint8, device=DEV)
    r = torch.full((P, P * b), 0xA5, dtype=torch.uint8, device=DEV)
    return s, r


def test_alltoall_errors(c):
    L, h, st = M.lib(), c.handle, _stream()
    s, r = _bufs(64)
    sp, rp = s.data_ptr(), r.data_ptr()
    for w in (0, 3, 5, 32):                                          # dtype_size
        _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_algo(sp, 1, w, rp, 0, h, st), r)
    _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_algo(None, 64, 1, rp, 0, h, st), r)      # NULL send
    _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_algo(sp, 64, 1, None, 0, h, st), r)      # NULL recv
    # overlap: recv inside send, and partially overlapping views of one buffer
    _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_algo(rp, 64, 1, rp, 0, h, st), r)
    _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_algo(rp + 100, 32, 1, rp, 0, h, st), r)
    _expect(c, M.ERR_ALGO, lambda: L.mpxa_alltoall_algo(sp, 64, 1, rp, M.ALGO["ring"], h, st), r)
    _expect(c, M.ERR_ALGO, lambda: L.mpxa_alltoall_algo(sp, 64, 1, rp, 99, h, st), r)
    _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_algo(sp, 64, 1, rp, 0, None, st), r)       # NULL comm
    # persistent form: the same checks at *_init, nothing bound
    q = ctypes.c_void_p()
    _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_init(rp, 64, 1, rp, 0, h, None, ctypes.byref(q)), r)
    _expect(c, M.ERR_ARG, lambda: L.mpxa_alltoall_init(sp, 16, 3, rp, 0, h, None, ctypes.byref(q)), r)
    _expect(c, M.ERR_ALGO, lambda: L.mpxa_alltoall_init(sp, 64, 1, rp, M.ALGO["ring"], h, None, ctypes.byref(q)), r)
    assert q.value is None


def test_allgather_errors(c):
    L, h, st = M.lib(), c.handle, _stream()
    s = torch.randint(0, 256, (P, 64), dtype=torch.uint8, device=DEV)
    r = torch.full((P, P * 64), 0xA5, dtype=torch.uint8, device=DEV)
    sp, rp = s.data_ptr(), r.data_ptr()
    _expect(c, M.ERR_ARG, lambda: L.mpxa_allgather_algo(sp, 1, 7, rp, 0, h, st), r)
    _expect(c, M.ERR_ARG, lambda: L.mpxa_allgather_algo(None, 64, 1, rp, 0, h, st), r)
    _expect(c, M.ERR_ARG, lambda: L.mpxa_allgather_algo(rp + 64, 64, 1, rp, 0, h, st), r)   # send inside recv
    _expect(c, M.ERR_ALGO, lambda: L.mpxa_allgather_algo(sp, 64, 1, rp, 77, h, st), r)
    q = ctypes.c_void_p()
    _expect(c, M.ERR_ARG, lambda: L.mpxa_allgather_init(sp, 64, 6, rp, 0, h, None, ctypes.byref(q)), r)
    _expect(c, M.ERR_ARG, lambda: L.mpxa_allgather_init(rp, 64, 1, rp, 0, h, None, ctypes.byref(q)), r)
    assert q.value is None


def _v_args(counts):
    sc = counts.astype(np.int64)
    rc = sc.T.copy()
    sd = np.zeros_like(sc)
    rd = np.zeros_like(rc)
    sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
    rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
    return sc, sd, rc, rd


def test_alltoallv_errors(c):
    counts = np.arange(P * P).reshape(P, P) % 5 + 1
    sc, sd, rc, rd = _v_args(counts)
    cap = 8 * int(max((sd + sc).max(), (rd + rc).max()))
    s = torch.randint(0, 256, (P, cap), dtype=torch.uint8, device=DEV)
    r = torch.full((P, cap), 0xA5, dtype=torch.uint8, device=DEV)

    def call(sc_=sc, sd_=sd, rc_=rc, rd_=rd, w=8, algo=None, send=s, recv=r):
        try:
            c.alltoallv(send, sc_, sd_, recv, rc_, rd_, algo=algo, dtype_size=w)
            return M.SUCCESS
        except MpxaError as e:
            return e.status

    def init(sc_=sc, rc_=rc, algo=None):
        try:
            c.alltoallv_init(s, sc_, sd, r, rc_, rd, algo=algo, dtype_size=8)
            return M.SUCCESS
        except MpxaError as e:
            return e.status

    neg = sc.copy()
    neg[1, 2] = -1
    _expect(c, M.ERR_ARG, lambda: call(sc_=neg), r)                         # negative count
    negd = rd.copy()
    negd[0, 0] = -8
    _expect(c, M.ERR_ARG, lambda: call(rd_=negd), r)                        # negative displacement
    big = rd.copy()
    big[3, 3] = cap // 8                                                    # displ + count > capacity
    _expect(c, M.ERR_ARG, lambda: call(rd_=big), r)
    bigs = sd.copy()
    bigs[2, 1] = cap // 8 - 1
    _expect(c, M.ERR_ARG, lambda: call(sd_=bigs), r)
    for w in (3, 6, 12):
        _expect(c, M.ERR_ARG, lambda: call(w=w), r)
    _expect(c, M.ERR_ARG, lambda: call(send=r), r)                          # overlap
    mis = rc.copy()
    mis[0, 1] += 1                                                          # sendcounts^T != recvcounts
    _expect(c, M.ERR_MISMATCH, lambda: call(rc_=mis), r)
    _expect(c, M.ERR_ALGO, lambda: call(algo="ring"), r)
    _expect(c, M.ERR_MISMATCH, lambda: init(rc_=mis), r)                    # persistent: at init
    _expect(c, M.ERR_ARG, lambda: init(sc_=neg), r)
    _expect(c, M.ERR_ALGO, lambda: init(algo="ring"), r)
    assert call() == M.SUCCESS                                              # the valid call still works
    torch.cuda.synchronize()
    assert c.check() == 0


def test_topology_errors():
    with pytest.raises(MpxaError) as e:                 # p = 4 ranks, groups of 3
        Comm(ranks_per_proc=4, device=0, group_size=3)
    assert e.value.status == M.ERR_TOPOLOGY
    with pytest.raises(MpxaError) as e:                 # 6 ranks over 4 emulated GPUs
        Comm(ranks_per_proc=6, device=0, emulate_gpus=4)
    assert e.value.status == M.ERR_TOPOLOGY
    with pytest.raises(MpxaError) as e:
        Comm(ranks_per_proc=0, device=0)
    assert e.value.status == M.ERR_TOPOLOGY


def test_lifecycle_and_registry_errors(c):
    s, r = _bufs(32)
    req = c.alltoall_init(s, r)
    with pytest.raises(MpxaError) as e:
        req.wait()                                      # wait on INACTIVE
    assert e.value.status == M.ERR_LIFECYCLE
    req.start()
    with pytest.raises(MpxaError) as e:
        req.start()                                     # start on ACTIVE
    assert e.value.status == M.ERR_LIFECYCLE
    with pytest.raises(MpxaError) as e:
        req.free()                                      # free while ACTIVE
    assert e.value.status == M.ERR_LIFECYCLE
    req.wait()
    req.free()
    with pytest.raises(MpxaError) as e:
        c.set_algorithm("alltoall", "ring")             # alltoall has no ring variant
    assert e.value.status == M.ERR_ALGO
    L = M.lib()
    out = ctypes.c_int()
    assert L.mpxa_get_algorithm(c.handle, 7, 64, ctypes.byref(out)) == M.ERR_ARG
    assert L.mpxa_load_selector(c.handle, b"/nonexistent/selector.txt") == M.ERR_ARG
    torch.cuda.synchronize()
    assert c.check() == 0

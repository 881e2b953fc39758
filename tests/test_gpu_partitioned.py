"""GPU tests of f3: partitioned point-to-point, -m gpu.

Parrived is compared with the oracle's byte-coverage predicate for the delivered sender
partitions (same and different receiver partitionings); every Pready order gives the
sender's bytes; 100 cycles with fresh data; the stream-ordered device Parrived holds a
consumer back until its partition has landed; a user producer kernel readies partitions
from the device (mpxa_dev_pready); lifecycle and matching errors."""
import ctypes
import itertools
import os
import subprocess

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2309_07337_b200 import Comm, MpxaError  # noqa: E402
from paper_2309_07337_b200 import mpxa as M  # noqa: E402

DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def channel(c, n_s, n_r, nbytes, src=0, dst=1, tag=0):
    s = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=DEV)
    r = torch.zeros(nbytes, dtype=torch.uint8, device=DEV)
    ps = c.psend_init(s, n_s, src, dst, tag)
    pr = c.precv_init(r, n_r, dst, src, tag)
    c.pmatch()
    return s, r, ps, pr


@pytest.mark.parametrize("n_s,n_r", [(4, 2), (4, 1), (4, 4), (3, 2), (2, 8), (1, 1)])
def test_parrived_matches_coverage_oracle(n_s, n_r):
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    nbytes = 48 * 1024
    s, r, ps, pr = channel(c, n_s, n_r, nbytes)
    rng = np.random.default_rng(n_s * 10 + n_r)
    for cyc in range(3):
        s.copy_(torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=DEV))
        pr.start()
        ps.start()
        delivered = np.zeros(n_s, np.uint8)
        for i in rng.permutation(n_s):
            torch.cuda.synchronize()
            want = oracle.part_arrived(n_s, nbytes // n_s, n_r, nbytes // n_r, delivered)
            assert [pr.parrived(j) for j in range(n_r)] == list(want), (cyc, delivered)
            ps.pready(int(i))
            delivered[i] = 1
        torch.cuda.synchronize()
        assert all(pr.parrived(j) for j in range(n_r))
        ps.wait()
        pr.wait()
        torch.cuda.synchronize()
        assert torch.equal(r, s)
        assert c.check() == 0
    ps.free(); pr.free()
    c.finalize()


def test_all_pready_orders_same_bytes():
    """every order of Pready over 4 partitions gives the sender's buffer."""
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    s, r, ps, pr = channel(c, 4, 2, 4096)
    for order in itertools.permutations(range(4)):
        r.zero_()
        s.copy_(torch.randint(0, 256, (4096,), dtype=torch.uint8, device=DEV))
        pr.start(); ps.start()
        for i in order:
            ps.pready(i)
        ps.wait(); pr.wait()
        torch.cuda.synchronize()
        assert torch.equal(r, s), order
    ps.free(); pr.free()
    c.finalize()


def test_hundred_cycles_large_partitions():
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    nbytes = 8 << 20
    s, r, ps, pr = channel(c, 8, 4, nbytes)
    l0 = c.launch_count()
    for cyc in range(100):
        if cyc in (0, 1, 99):
            s.copy_(torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=DEV))
        pr.start(); ps.start()
        ps.pready(0, 8)
        ps.wait(); pr.wait()
        if cyc in (0, 1, 99):
            torch.cuda.synchronize()
            assert torch.equal(r, s), cyc
    assert c.launch_count() - l0 == 100 * 5          # start x2, pready, wait x2: no setup per cycle
    ps.free(); pr.free()
    c.finalize()


@pytest.mark.parametrize("n_s,n_r", [(16, 4), (4, 16)])
def test_256MiB_channel_producer_on_other_stream(n_s, n_r):
    """The bench's f3 point at full size (256 MiB, 16->4 and 4->16), 10 cycles.  Every cycle
    the producer fills the send buffer on ITS OWN stream and the channel stream waits on an
    event recorded after the fill (stream-ordered readiness); the receiver
    buffer is re-zeroed the same way.  Whole-buffer byte equality (SPEC.md's byte-equality
    oracle) plus Parrived of every receiver partition against the coverage oracle."""
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    nbytes = 256 << 20
    prod, chan = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(prod):
        s = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
        r = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    torch.cuda.synchronize()
    ps = c.psend_init(s, n_s, 0, 1)
    pr = c.precv_init(r, n_r, 1, 0)
    c.pmatch()
    gen = torch.Generator(device=DEV)
    for cyc in range(10):
        gen.manual_seed(77 + cyc)
        with torch.cuda.stream(prod):
            s.random_(0, 256, generator=gen)
            r.zero_()
            ev = torch.cuda.Event()
            ev.record(prod)
        chan.wait_event(ev)
        pr.start(chan); ps.start(chan)
        ps.pready(0, n_s, stream=chan)
        ps.wait(chan)
        chan.synchronize()
        ones = np.ones(n_s, np.uint8)
        assert [pr.parrived(j) for j in range(n_r)] == list(oracle.part_arrived(n_s, nbytes // n_s, n_r,
                                                                                 nbytes // n_r, ones))
        pr.wait(chan)
        chan.synchronize()
        assert torch.equal(r, s), cyc
        prod.wait_stream(chan)      # next fill only after this cycle's reads of s / writes of r
    assert c.check() == 0
    ps.free(); pr.free()
    c.finalize()


def test_large_pready_ranges_out_of_order():
    """Host Pready calls of >= 64 MiB take the TMA slice kernel (several waves of short
    slices); ranges readied out of order and one partition at a time (p0 > 0) deliver the
    same bytes, and Parrived follows the coverage oracle after each call."""
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    nbytes, n_s, n_r = 256 << 20, 4, 8
    s = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    r = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    ps = c.psend_init(s, n_s, 0, 1)
    pr = c.precv_init(r, n_r, 1, 0)
    c.pmatch()
    gen = torch.Generator(device=DEV)
    for cyc, order in enumerate(([(2, 4), (0, 2)], [(3, 4), (1, 2), (0, 1), (2, 3)])):
        gen.manual_seed(5 + cyc)
        s.random_(0, 256, generator=gen)
        r.zero_()
        torch.cuda.synchronize()
        pr.start(); ps.start()
        ready = np.zeros(n_s, np.uint8)
        for lo, hi in order:
            ps.pready(lo, hi)
            torch.cuda.synchronize()
            ready[lo:hi] = 1
            want = oracle.part_arrived(n_s, nbytes // n_s, n_r, nbytes // n_r, ready)
            assert [pr.parrived(j) for j in range(n_r)] == list(want), (cyc, lo, hi)
        ps.wait(); pr.wait()
        torch.cuda.synchronize()
        assert torch.equal(r, s), cyc
    assert c.check() == 0
    ps.free(); pr.free()
    c.finalize()


def test_device_parrived_orders_consumer_after_arrival():
    """mpxa_parrived_wait on the consumer stream: the copy behind it sees partition 0 even
    though the sender readies it only after a long device delay on another stream."""
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    nbytes = 1 << 20
    s, r, ps, pr = channel(c, 2, 2, nbytes)
    prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
    out = torch.zeros(nbytes // 2, dtype=torch.uint8, device=DEV)
    pr.start(cons); ps.start(prod)
    torch.cuda.synchronize()
    with torch.cuda.stream(prod):
        torch.cuda._sleep(200_000_000)               # ~0.1 s of device time before Pready
        ps.pready(0, stream=prod)
    pr.parrived_wait(0, stream=cons)
    with torch.cuda.stream(cons):
        out.copy_(r[: nbytes // 2])
    ps.pready(1, stream=prod)
    ps.wait(prod); pr.wait(cons)
    torch.cuda.synchronize()
    assert torch.equal(out, s[: nbytes // 2])
    ps.free(); pr.free()
    c.finalize()


def test_device_side_pready_from_producer_kernel(tmp_path):
    """Early-bird from the device: a user kernel computes each partition and readies it with
    mpxa_dev_pready (include/mpxa_device.cuh)."""
    so = tmp_path / "producer.so"
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                           "-shared", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cuda", "producer.cu"), "-o", str(so)])
    lib = ctypes.CDLL(str(so))
    lib.launch_produce.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    n_s, nbytes = 16, 16 * 65536
    s, r, ps, pr = channel(c, n_s, 4, nbytes)
    for seed in (1, 2):
        pr.start(); ps.start()
        h = ps.device_handle()
        assert lib.launch_produce(h, n_s, s.data_ptr(), seed, torch.cuda.current_stream().cuda_stream) == 0
        ps.wait(); pr.wait()
        torch.cuda.synchronize()
        k = np.arange(65536)
        want = np.concatenate([((k * 131 + i * 7 + seed) & 0xFF).astype(np.uint8) for i in range(n_s)])
        assert np.array_equal(r.cpu().numpy(), want), seed
    ps.free(); pr.free()
    c.finalize()


def test_partitioned_errors():
    c = Comm(ranks_per_proc=2, device=0, timeout_s=20.0)
    s = torch.zeros(1024, dtype=torch.uint8, device=DEV)
    r = torch.zeros(1024, dtype=torch.uint8, device=DEV)
    ps = c.psend_init(s, 4, 0, 1, 5)
    with pytest.raises(MpxaError) as e:            # no receiver yet: the single match fails
        c.pmatch()
    assert e.value.status == M.ERR_MISMATCH
    r2 = torch.zeros(512, dtype=torch.uint8, device=DEV)
    pr_bad = c.precv_init(r2, 2, 1, 0, 5)
    with pytest.raises(MpxaError) as e:            # total bytes differ
        c.pmatch()
    assert e.value.status == M.ERR_MISMATCH
    pr_bad.free()
    pr = c.precv_init(r, 2, 1, 0, 5)
    c.pmatch()
    with pytest.raises(MpxaError) as e:            # pready before start
        ps.pready(0)
    assert e.value.status == M.ERR_LIFECYCLE
    pr.start(); ps.start()
    ps.pready(1)
    with pytest.raises(MpxaError) as e:            # twice in one cycle
        ps.pready(1)
    assert e.value.status == M.ERR_ARG
    with pytest.raises(MpxaError) as e:            # out of range
        ps.pready(4)
    assert e.value.status == M.ERR_ARG
    ps.pready(0); ps.pready(2, 4)
    ps.wait(); pr.wait()
    with pytest.raises(MpxaError) as e:            # wait on INACTIVE
        pr.wait()
    assert e.value.status == M.ERR_LIFECYCLE
    with pytest.raises(MpxaError):
        c.psend_init(s, 4, 5, 1, 0)                 # rank not hosted here
    torch.cuda.synchronize()
    assert torch.equal(r, s)
    ps.free(); pr.free()
    c.finalize()


def test_watchdog_poisons_comm_on_missing_partition():
    """SURVEY.md §5 failure detection: a partition never readied makes the receiver's device
    wait time out; the error word maps to MPXA_ERR_TIMEOUT and the comm is poisoned (no hang)."""
    c = Comm(ranks_per_proc=2, device=0, timeout_s=0.3)
    s, r, ps, pr = channel(c, 4, 4, 4096)
    pr.start(); ps.start()
    ps.pready(0, 3)                                 # partition 3 is never readied
    pr.wait()
    torch.cuda.synchronize()
    assert c.check() == M.ERR_TIMEOUT
    with pytest.raises(MpxaError) as e:
        pr.start()
    assert e.value.status == M.ERR_TIMEOUT
    with pytest.raises(MpxaError) as e:             # collectives refuse to run on a poisoned comm
        x = torch.zeros(2 * 2 * 64, dtype=torch.uint8, device=DEV)
        c.alltoall(x, torch.empty_like(x))
    assert e.value.status == M.ERR_TIMEOUT

"""B1, the NCCL baseline, checked bit-exactly against the oracle (-m gpu).

NCCL's grouped ncclSend/ncclRecv alltoall(v) and ncclAllGather, called from C++
(baseline/b1), must produce exactly the oracle's definitions on the same seeded inputs --
"NCCL output is also checked bit-exactly against the oracle".  One
process per visible GPU (one NCCL rank per GPU); the single-GPU case is a 1-rank
communicator (self send/recv), the multi-GPU case is skipped below 2 GPUs."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import mp_util  # noqa: E402


def _body(rank, world):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import oracle
    import synth
    from baseline import b1 as B1
    torch.cuda.set_device(rank)
    dev = f"cuda:{rank}"
    B1.build()
    nc = B1.NcclB1(dist.group.WORLD, rank)
    p = world
    for b in (4, 1000, 65536 + 12, 1 << 20):
        # alltoall: recv_r[j] = send_j[r]
        send_all = synth.alltoall_sendbuf(b, p, b)
        want = oracle.alltoall_definition(send_all)
        s = torch.from_numpy(send_all[rank].copy()).to(dev)
        r = torch.full((p * b,), 0xA5, dtype=torch.uint8, device=dev)
        nc.call("alltoall", s, r, b)
        torch.cuda.synchronize()
        assert np.array_equal(r.cpu().numpy(), want[rank]), ("alltoall", b)
        # allgather, both forms
        ag = synth.allgather_sendbuf(b, p, b)
        agw = oracle.allgather_definition(ag)
        s = torch.from_numpy(ag[rank].copy()).to(dev)
        for op in ("allgather", "allgather_grouped"):
            r = torch.full((p * b,), 0x5A, dtype=torch.uint8, device=dev)
            nc.call(op, s, r, b)
            torch.cuda.synchronize()
            assert np.array_equal(r.cpu().numpy(), agw[rank]), (op, b)
    # alltoallv, cfg4 counts (int64 elements) with gaps between received segments
    counts = synth.cfg4_counts(0, p, 64 << 10)
    send_all, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, counts, elem=8, packed=False)
    recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send_all, sc, sd, rc, rd, 8, recv0)
    s = torch.from_numpy(send_all[rank].copy()).to(dev)
    r = torch.from_numpy(recv0[rank].copy()).to(dev)
    nc.call("alltoallv", s, r, v=(sc[rank] * 8, sd[rank] * 8, rc[rank] * 8, rd[rank] * 8))
    torch.cuda.synchronize()
    assert np.array_equal(r.cpu().numpy(), want[rank]), "alltoallv"
    # the timing entry points run (events and CUDA-graph modes)
    s = torch.empty(p * 4096, dtype=torch.uint8, device=dev)
    r = torch.empty_like(s)
    assert nc.time("alltoall", s, r, 4096, warmup=2, iters=10, graph=True) > 0
    assert nc.time("allgather", s[:4096], r, 4096, warmup=2, iters=10, graph=False) > 0
    nc.finalize()


def test_b1_one_rank_vs_oracle():
    mp_util.spawn(_body, 1)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (one NCCL rank per GPU)")
def test_b1_all_gpus_vs_oracle():
    mp_util.spawn(_body, torch.cuda.device_count())

"""GPU parity of f1: persistent neighborhood alltoallv, standard and locality-aware
(SPEC.md:297-325), through the C ABI on sm_100a, bit-exact against the
oracle (-m gpu).  All ranks on one device, also split over emulated GPUs (multi-GPU flag
protocol), locality groups of 1, 2 and R ranks; canaries outside received ranges must
survive; 100 start/wait cycles with fresh data; the one-shot call."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2309_07337_b200 import Comm, MpxaError  # noqa: E402
from paper_2309_07337_b200 import mpxa as M  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def per_rank_lists(p, gr):
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])])
    ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
    srcs = [list(map(int, gr["src"][ioff[r]:ioff[r + 1]])) for r in range(p)]
    dsts = [list(map(int, gr["dst"][ooff[r]:ooff[r + 1]])) for r in range(p)]
    return srcs, dsts


def cases():
    yield "ring", 4, synth.ring_edges(4, 5)
    yield "stencil9", 8, synth.stencil_edges(4, 2, 64, 32, corners=True)
    yield "spmv", 8, synth.spmv_edges(3, 8, 64, 24, 3)
    yield "random", 8, synth.random_edges(11, 8, 5, 40, 60)
    yield "empty", 4, []


@pytest.mark.parametrize("name,p,edges", list(cases()), ids=[c[0] for c in cases()])
def test_neighbor_parity(name, p, edges):
    gr, si, ri = synth.graph_from_edges(p, edges)
    send, recv0 = synth.neighbor_buffers(7, p, gr, si, w=8)
    want = oracle.neighbor_definition(send, recv0, 8, gr)
    srcs, dsts = per_rank_lists(p, gr)
    for G in [0] + [G for G in (2, 4) if p % G == 0]:
        for g in [x for x in (1, 2, p) if p % x == 0]:
            c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=g, timeout_s=20.0)
            topo = c.dist_graph_create_adjacent(srcs, dsts)
            for loc in (False, True):
                d_send, d_recv = dev(send), dev(recv0)
                kw = dict(send_indices=si, recv_indices=ri) if loc else {}
                req = c.neighbor_alltoallv_init(topo, d_send, gr["sc"], gr["sd"], d_recv, gr["rc"], gr["rd"],
                                                dtype_size=8, **kw)
                assert req.algorithm == ("locality" if loc else "pairwise")
                req.start()
                req.wait()
                assert np.array_equal(host(d_recv), want), (name, G, g, loc)
                assert c.check() == 0
                req.free()
            topo.free()
            c.finalize()


def test_neighbor_persistent_cycles_and_one_shot():
    p = 8
    gr, si, ri = synth.graph_from_edges(p, synth.spmv_edges(5, p, 256, 96, 3))
    srcs, dsts = per_rank_lists(p, gr)
    for G in (0, 4):
        c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=2, timeout_s=20.0)
        topo = c.dist_graph_create_adjacent(srcs, dsts)
        send0, recv0 = synth.neighbor_buffers(0, p, gr, si, w=8)
        d_send, d_recv = dev(send0), dev(recv0)
        req = c.neighbor_alltoallv_init(topo, d_send, gr["sc"], gr["sd"], d_recv, gr["rc"], gr["rd"], dtype_size=8,
                                        send_indices=si, recv_indices=ri)
        l0 = c.launch_count()
        for cyc in range(100):
            if cyc in (0, 1, 99):
                send_c, _ = synth.neighbor_buffers(100 + cyc, p, gr, si, w=8)
                d_send.copy_(dev(send_c))
            req.start()
            req.wait()
            if cyc in (0, 1, 99):
                assert np.array_equal(host(d_recv), oracle.neighbor_definition(send_c, recv0, 8, gr)), (G, cyc)
        assert c.launch_count() - l0 == 100                # init once; one kernel per start
        req.free()
        # one-shot standard call
        send1, _ = synth.neighbor_buffers(9, p, gr, si, w=8)
        d_recv2 = dev(recv0)
        c.neighbor_alltoallv(topo, dev(send1), gr["sc"], gr["sd"], d_recv2, gr["rc"], gr["rd"], dtype_size=8)
        assert np.array_equal(host(d_recv2), oracle.neighbor_definition(send1, recv0, 8, gr))
        topo.free()
        c.finalize()


def test_neighbor_errors():
    p = 4
    c = Comm(ranks_per_proc=p, device=0, group_size=2)
    gr, si, ri = synth.graph_from_edges(p, [(0, 2, [7, 8]), (1, 3, [9])])
    srcs, dsts = per_rank_lists(p, gr)
    topo = c.dist_graph_create_adjacent(srcs, dsts)
    send, recv0 = synth.neighbor_buffers(0, p, gr, si)
    d_send, d_recv = dev(send), dev(recv0)
    bad = gr["rc"].copy()
    bad[0] += 1
    with pytest.raises(MpxaError) as e:
        c.neighbor_alltoallv_init(topo, d_send, gr["sc"], gr["sd"], d_recv, bad, gr["rd"], dtype_size=8)
    assert e.value.status in (M.ERR_MISMATCH, M.ERR_ARG)
    wrong = ri.copy()
    wrong[0] = 99
    with pytest.raises(MpxaError) as e:
        c.neighbor_alltoallv_init(topo, d_send, gr["sc"], gr["sd"], d_recv, gr["rc"], gr["rd"], dtype_size=8,
                                  send_indices=si, recv_indices=wrong)
    assert e.value.status == M.ERR_TOPOLOGY
    with pytest.raises(MpxaError) as e:
        c.dist_graph_create_adjacent([[9]] + [[]] * 3, [[]] * 4)    # rank out of range
    assert e.value.status == M.ERR_ARG
    topo.free()
    c.finalize()

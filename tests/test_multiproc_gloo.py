"""World-size-2 gloo tests of the multi-process host logic (-m "not gpu").

Each process plays one GPU of a 2-GPU communicator:
  * the bootstrap all-gather callback libmpxa calls during collective setup (Python,
    over gloo) returns every process's bytes in process order;
  * each process all-gathers the count/displacement rows (as mpxa_alltoallv does in
    multi-process mode), builds the GLOBAL schedule itself, and executes only the moves its
    GPU owns; remote writes travel to the peer over gloo.  The composed result must equal
    the oracle, and both processes must have compiled the identical schedule.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WS = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(rank, port, fn, q):  # noqa: C901
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        fn(rank)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def spawn(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, port, fn, q)) for r in range(WS)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, msg in res:
        assert msg == "ok", f"rank {r}: {msg}"


# --------------------------------------------------------------------------------------

def _bootstrap_body(rank):
    import ctypes
    from paper_2309_07337_b200.mpxa import make_bootstrap
    cb = make_bootstrap(dist.group.WORLD, WS)
    n = 24
    inp = (ctypes.c_uint8 * n)(*[(rank * 31 + i) % 256 for i in range(n)])
    out = (ctypes.c_uint8 * (n * WS))()
    assert cb(ctypes.addressof(inp), ctypes.addressof(out), n, None) == 0
    got = bytes(out)
    for r in range(WS):
        assert got[r * n:(r + 1) * n] == bytes((r * 31 + i) % 256 for i in range(n))


def test_bootstrap_allgather_callback():
    spawn(_bootstrap_body)


def _sim_body(rank):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle
    import synth
    from paper_2309_07337_b200 import Plan

    SEND, RECV, WORK = 0, 1, 2
    R = 4                          # ranks per process ("GPU")
    p = R * WS
    for case in ("alltoall_pairwise", "alltoall_bruck", "alltoall_hier", "allgather_ring",
                 "allgather_bruck", "allgather_pairwise", "alltoallv_pairwise", "alltoallv_hier"):
        op, algo = case.split("_")
        unit = 3 if op != "alltoallv" else 8
        counts = sd = rd = None
        if op == "alltoall":
            send_all = synth.alltoall_sendbuf(5, p, unit)
            want = oracle.alltoall_definition(send_all)
        elif op == "allgather":
            send_all = synth.allgather_sendbuf(5, p, unit)
            want = oracle.allgather_definition(send_all)
        else:
            c = synth.cfg4_counts(3, p, 32)
            send_all, sc, sdl, rc, rdl, S, Rcap = synth.alltoallv_buffers(3, c, elem=8, packed=False)
            # this process only knows ITS rows; all-gather them like mpxa_alltoallv does
            mine = np.stack([sc[rank * R:(rank + 1) * R], sdl[rank * R:(rank + 1) * R],
                             rc[rank * R:(rank + 1) * R], rdl[rank * R:(rank + 1) * R]])
            allrows = [None] * WS
            dist.all_gather_object(allrows, mine)
            counts = np.concatenate([a[0] for a in allrows])
            sd = np.concatenate([a[1] for a in allrows])
            rd = np.concatenate([a[3] for a in allrows])
            assert np.array_equal(counts, sc) and np.array_equal(np.concatenate([a[2] for a in allrows]), rc)
            recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
            want = oracle.alltoallv_definition(send_all, sc, sdl, rc, rdl, 8, recv0)
        pl = Plan(op, algo, p, R=R, G=WS, g=R, counts=counts, sdispls=sd, rdispls=rd)
        # identical schedule on every process
        sig = [(m.src_kind, m.src_rank, m.src_off, m.dst_kind, m.dst_rank, m.dst_off, m.len, m.flow)
               for g in range(WS) for m in pl.moves(g)]
        sigs = [None] * WS
        dist.all_gather_object(sigs, hash(tuple(sig)))
        assert sigs[0] == sigs[1]
        # my buffers only (rows of my ranks); peers' rows are not present here
        send = send_all.copy()
        recv = np.full_like(want, 0xA5) if op == "alltoallv" else np.zeros_like(want)
        work = np.zeros((p, max(1, pl.info["work_units"]) * unit), dtype=np.uint8)
        bufs = {SEND: send, RECV: recv, WORK: work}
        mine_ranks = range(rank * R, (rank + 1) * R)
        steps = pl.steps(rank)
        moves = pl.moves(rank)
        for s, st in enumerate(steps):
            remote = []
            local = []
            for m in moves[st.move_begin:st.move_end]:
                assert m.src_rank in mine_ranks
                data = bufs[m.src_kind][m.src_rank, m.src_off * unit:(m.src_off + m.len) * unit].copy()
                for d in (range(p) if m.fanout else [m.dst_rank]):
                    item = (m.dst_kind, d, m.dst_off * unit, data)
                    (local if d in mine_ranks else remote).append(item)
                    if d not in mine_ranks:
                        assert (st.signal_mask >> (d // R)) & 1
            got = [None] * WS
            dist.all_gather_object(got, remote)
            incoming = [it for r, lst in enumerate(got) if r != rank for it in lst if it[1] in mine_ranks]
            if incoming:
                assert (st.wait_mask >> (1 - rank)) & 1
            for k, d, o, data in local + incoming:
                bufs[k][d, o:o + len(data)] = data
        rows = slice(rank * R, (rank + 1) * R)
        assert np.array_equal(recv[rows], want[rows]), case


def test_two_process_schedule_composition():
    spawn(_sim_body)


# --------------------------------------------------------------------------------------
# cross-process configuration consistency (mpxa_init, before any CUDA call)

def _knob_body(rank, cases):
    """Each case: (env of rank 0, env of rank 1, expected); all cases run in order on both
    processes (mpxa_init is collective)."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2309_07337_b200 import Comm, MpxaError
    from paper_2309_07337_b200 import mpxa as M
    for env_by_rank, expect in cases:
        env = env_by_rank[rank]
        for k, v in env.items():
            os.environ[k] = v
        try:
            c = Comm(ranks_per_proc=2, device=0, pg=dist.group.WORLD, timeout_s=5.0)
            status = M.SUCCESS
            c.finalize()
        except MpxaError as e:
            status = e.status
        for k in env:
            del os.environ[k]
        # equal configurations pass the check and init proceeds to the device (no GPU here:
        # MPXA_ERR_CUDA; on a GPU box it may succeed); unequal ones stop at the check
        if expect == "mismatch":
            assert status == M.ERR_MISMATCH, (env_by_rank, status)
        else:
            assert status in (M.SUCCESS, M.ERR_CUDA), (env_by_rank, status)


def test_init_knob_consistency(tmp_path):
    """processes that disagree on a protocol knob, the selector table or a forced
    variant must fail mpxa_init with MPXA_ERR_MISMATCH (on every process), not desynchronize
    the eager / direct protocols at the first launch."""
    import functools
    sel = tmp_path / "sel.txt"
    sel.write_text("alltoall 4 2 1024 bruck\n")
    cases = [([{}, {k: v}], "mismatch") for k, v in (
        ("MPXA_NO_LL", "1"),                  # eager protocol on one process only
        ("MPXA_LL_MAX", "4096"),
        ("MPXA_ROW_SIGNAL", "0"),
        ("MPXA_HIER_STAGED", "1"),
        ("MPXA_ALGO", "alltoall:bruck"),
        ("MPXA_NO_SMALL", "1"),
        ("MPXA_NO_WRING", "1"),                # warp-ring dynamic mode on one process only
        ("MPXA_SMALL_ITEMS", "2048"),          # small-kernel grid (CTA flag slots pair 1:1)
        ("MPXA_OWN_VOL", "1048576"),            # owned-flow vs row-barrier mode
        ("MPXA_SELECTOR", str(sel)))]
    same = {"MPXA_NO_LL": "1", "MPXA_SELECTOR": str(sel)}
    cases += [([same, dict(same)], "ok"), ([{}, {}], "ok")]
    spawn(functools.partial(_knob_body, cases=cases))

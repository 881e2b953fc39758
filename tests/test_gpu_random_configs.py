"""Randomized differential tests (-m gpu): seeded random collectives -- op, variant, rank
count, emulated GPU split, block / count sizes, dtype size, buffer misalignment, persistent
or one-shot -- each checked bit-exactly against the oracle with canaries around the results.
Covers the launch-path combinations the directed tests reach one at a time (small kernel
modes, eager staging, variable pieces, shared-memory WORK, block sizing, executor)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2309_07337_b200 import Comm

pytestmark = pytest.mark.gpu
DEV = "cuda"
_COMMS = {}


def comm(p, G, g):
    key = (p, G, g)
    if key not in _COMMS:
        _COMMS[key] = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=g, timeout_s=20.0)
    return _COMMS[key]


def splits(p):
    return [0] + [G for G in (2, 3, 4, 8) if p % G == 0 and G <= p]


def to_dev(a, off):
    """uint8 rows -> device buffer shifted by `off` bytes (misaligned base), plus the view."""
    flat = torch.zeros(a.size + 64, dtype=torch.uint8, device=DEV)
    flat[off:off + a.size] = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(DEV)
    return flat, flat[off:off + a.size].view(a.shape)


@pytest.mark.parametrize("seed", range(int(os.environ.get("MPXA_RANDOM_SEEDS", "96"))))
def test_random_alltoall_allgather(seed):
    rng = np.random.default_rng(1000 + seed)
    p = int(rng.choice([2, 3, 4, 6, 8, 12, 16]))
    G = int(rng.choice(splits(p)))
    g = int(rng.choice([x for x in (1, 2, 3, 4) if p % x == 0]))
    b = int(rng.choice([1, 3, 8, 16, 44, 256, 1000, 4096, 4100, 65536, 70000, 300_000, 1 << 20]))
    if p * p * b > (48 << 20):   # keep the executor-sized draws to small p
        b = 70000
    off = int(rng.choice([0, 0, 1, 4, 8]))
    c = comm(p, G, g)
    send = rng.integers(0, 256, size=(p, p * b), dtype=np.uint8)
    want = oracle.alltoall_definition(send)
    _, d_s = to_dev(send, off)
    canary = np.full((p, p * b), 0xC3, np.uint8)
    keep_r, d_r = to_dev(canary, (off * 3) % 16)
    algo = str(rng.choice(["pairwise", "bruck", "hier"]))
    if rng.random() < 0.3:
        req = c.alltoall_init(d_s, d_r, algo=algo)
        for _ in range(int(rng.integers(1, 4))):
            req.start(); req.wait()
        req.free()
    else:
        c.alltoall(d_s, d_r, algo=algo)
    torch.cuda.synchronize()
    assert np.array_equal(d_r.cpu().numpy(), want), (p, G, g, b, off, algo)
    # allgather on the same comm
    ag = rng.integers(0, 256, size=(p, b), dtype=np.uint8)
    _, d_a = to_dev(ag, off)
    keep_o, d_o = to_dev(np.full((p, p * b), 0x3C, np.uint8), 0)
    algo = str(rng.choice(["pairwise", "bruck", "ring", "hier"]))
    c.allgather(d_a, d_o, algo=algo)
    torch.cuda.synchronize()
    assert np.array_equal(d_o.cpu().numpy(), oracle.allgather_definition(ag)), (p, G, b, algo)
    assert c.check() == 0


@pytest.mark.parametrize("seed", range(int(os.environ.get("MPXA_RANDOM_SEEDS", "96")) * 2 // 3))
def test_random_alltoallv(seed):
    rng = np.random.default_rng(2000 + seed)
    p = int(rng.choice([2, 4, 5, 8, 16]))
    G = int(rng.choice(splits(p)))
    g = int(rng.choice([x for x in (1, 2, 4) if p % x == 0]))
    w = int(rng.choice([1, 2, 4, 8, 16]))
    shape = rng.choice(["tiny", "mixed", "mid"])
    if shape == "tiny":
        counts = rng.integers(0, 5, size=(p, p))
    elif shape == "mixed":
        counts = rng.integers(0, 3, size=(p, p))
        big = rng.choice(p * p, size=max(1, p // 2), replace=False)
        counts.reshape(-1)[big] = rng.integers(2000, 9000, size=big.size)
    else:
        counts = rng.integers(0, 3000, size=(p, p))
    counts[rng.random((p, p)) < 0.1] = 0
    counts = counts.astype(np.int64)
    sc, rc = counts, counts.T.copy()
    gs, gr = rng.integers(0, 3, size=(p, p)), rng.integers(0, 3, size=(p, p))
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc + gs, 1)[:, :-1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc + gr, 1)[:, :-1]
    S = int((sd + sc).max()) + 4
    R = int((rd + rc).max()) + 4
    send = rng.integers(0, 256, size=(p, S * w), dtype=np.uint8)
    recv0 = np.full((p, R * w), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, w, recv0)
    c = comm(p, G, g)
    algo = str(rng.choice(["pairwise", "hier", "bruck"]))
    d_s = torch.from_numpy(send).to(DEV)
    d_r = torch.from_numpy(recv0).to(DEV)
    if rng.random() < 0.4:
        req = c.alltoallv_init(d_s, sc, sd, d_r, rc, rd, algo=algo, dtype_size=w)
        for _ in range(int(rng.integers(1, 4))):
            req.start(); req.wait()
        req.free()
    else:
        c.alltoallv(d_s, sc, sd, d_r, rc, rd, algo=algo, dtype_size=w)
    torch.cuda.synchronize()
    assert np.array_equal(d_r.cpu().numpy(), want), (p, G, g, w, shape, algo)
    assert c.check() == 0


KNOBS = [{"MPXA_NO_LL": "1"}, {"MPXA_NO_SMALL": "1"}, {"MPXA_NO_DYN": "1"}, {"MPXA_SWORK": "0"},
         {"MPXA_SMALL_NT": "512"}, {"MPXA_NO_PDL": "1"}, {"MPXA_NO_SMALL_SYNC": "1"},
         {"MPXA_HIER_STAGED": "1"}, {"MPXA_ROW_SIGNAL": "0", "MPXA_NO_SMALL": "1"},
         # every dynamic launch through the per-warp TMA rings, multi-step programs included
         {"MPXA_WRING": "2", "MPXA_DYN_SYNC": "1", "MPXA_NO_SMALL": "1"},
         # the general small kernel for launches the tiny kernels would take
         {"MPXA_NO_TINY": "1"},
         # the round-2 grid sizing choices, reverted: power-of-two tiny blocks, 2048 pieces per
         # small-kernel CTA, the smaller owned-flow limits
         {"MPXA_TINY_EVEN": "0"}, {"MPXA_SMALL_ITEMS": "2048"},
         {"MPXA_OWN_VOL": "2097152", "MPXA_OWN_PER_CTA": "65536"},
         # no pre-wait L2 prefetch of the dynamic mode's first pieces
         {"MPXA_NO_PREFETCH": "1", "MPXA_NO_SMALL": "1"}]


@pytest.mark.parametrize("knob", range(len(KNOBS)), ids=[",".join(k) for k in KNOBS])
def test_random_under_path_knobs(knob, monkeypatch):
    """The same random draws with a launch-path knob forcing the alternative path (direct
    instead of eager, executor instead of small kernel, static slices instead of queues, ...):
    every path stays exact."""
    for k, v in KNOBS[knob].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(3000 + knob)
    for it in range(6):
        p = int(rng.choice([3, 4, 8]))
        G = int(rng.choice(splits(p)))
        g = int(rng.choice([x for x in (1, 2, 4) if p % x == 0]))
        b = int(rng.choice([1, 16, 100, 4096, 70000]))
        c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=g, timeout_s=20.0)
        send = rng.integers(0, 256, size=(p, p * b), dtype=np.uint8)
        d_r = torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
        algo = str(rng.choice(["pairwise", "bruck", "hier"]))
        c.alltoall(torch.from_numpy(send).to(DEV), d_r, algo=algo)
        torch.cuda.synchronize()
        assert np.array_equal(d_r.cpu().numpy(), oracle.alltoall_definition(send)), (knob, p, G, b, algo)
        ag = rng.integers(0, 256, size=(p, b), dtype=np.uint8)
        d_o = torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
        algo = str(rng.choice(["pairwise", "bruck", "ring"]))
        c.allgather(torch.from_numpy(ag).to(DEV), d_o, algo=algo)
        torch.cuda.synchronize()
        assert np.array_equal(d_o.cpu().numpy(), oracle.allgather_definition(ag)), (knob, p, G, b, algo)
        assert c.check() == 0
        c.finalize()

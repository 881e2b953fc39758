"""Eager (LL) schedules (mpxa_plan_eager; SURVEY.md §8 A9 "epoch-parity staging for eager
mode") simulated on the CPU (-m "not gpu"): for every multi-GPU split, variant and a few
unit sizes, the eager form of the plan must reproduce the oracle bit for bit, keep its
receives last in each step, write every staging word once and only read it after it was
written, and make every ordered GPU pair exchange at least one word."""
import numpy as np
import pytest

import oracle
import synth
from paper_2309_07337_b200 import Plan, MpxaError
from paper_2309_07337_b200 import mpxa as M
from plan_sim import simulate_eager, LL_WORDS


def splits(p):
    return [G for G in range(2, p + 1) if p % G == 0]


@pytest.mark.parametrize("p", [2, 3, 4, 6, 8])
@pytest.mark.parametrize("algo", ["pairwise", "bruck", "hier"])
def test_eager_alltoall_plans(p, algo):
    for b in (1, 4, 13, 64):
        send = synth.alltoall_sendbuf(b + p, p, b)
        want = oracle.alltoall_definition(send)
        for G in splits(p):
            g = 2 if p % 2 == 0 else 1
            pl = Plan("alltoall", algo, p, G=G, g=g)
            e = pl.eager(b)
            got = simulate_eager(e, send, np.zeros_like(send), b)
            assert np.array_equal(got, want), (p, G, b, algo)


@pytest.mark.parametrize("p", [2, 4, 5, 8])
@pytest.mark.parametrize("algo", ["pairwise", "bruck", "ring", "hier"])
def test_eager_allgather_plans(p, algo):
    if algo == "hier" and p % 2:
        return
    for b in (1, 7, 32):
        ag = np.random.default_rng(b).integers(0, 256, size=(p, b), dtype=np.uint8)
        want = oracle.allgather_definition(ag)
        for G in splits(p):
            pl = Plan("allgather", algo, p, G=G, g=2 if algo == "hier" else 1)
            got = simulate_eager(pl.eager(b), ag, np.zeros((p, p * b), np.uint8), b)
            assert np.array_equal(got, want), (p, G, b, algo)


def test_eager_alltoallv_sparse_pairs():
    """Most GPU pairs exchange nothing: one flag word each (len 0); canaries untouched."""
    p = 8
    counts = np.zeros((p, p), np.int64)
    counts[0, 5], counts[3, 3], counts[6, 1], counts[7, 7] = 37, 11, 4, 9
    sc, rc = counts, counts.T.copy()
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
    S, R = int((sd + sc).max()) + 8, int((rd + rc).max()) + 8
    rng = np.random.default_rng(3)
    send = rng.integers(0, 256, size=(p, S), dtype=np.uint8)
    recv0 = np.full((p, R), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 1, recv0)
    for G in (2, 4, 8):
        for algo in ("pairwise", "hier", "bruck"):
            pl = Plan("alltoallv", algo, p, G=G, g=2, counts=sc, sdispls=sd, rdispls=rd)
            e = pl.eager(1)
            assert np.array_equal(simulate_eager(e, send, recv0, 1), want), (G, algo)


def test_eager_ineligible():
    """Single GPU, or a GPU pair needing more than the staging holds -> ERR_ALGO."""
    with pytest.raises(MpxaError) as e:
        Plan("alltoall", "pairwise", 4, G=1).eager(16)
    assert e.value.status == M.ERR_ALGO
    with pytest.raises(MpxaError) as e:
        Plan("alltoall", "pairwise", 4, G=4).eager(4 * LL_WORDS + 4)
    assert e.value.status == M.ERR_ALGO
    Plan("alltoall", "pairwise", 4, G=4).eager(4 * LL_WORDS)     # exactly full: fine

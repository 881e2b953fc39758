"""CPU tests of the product's host side (-m "not gpu"): the C ABI loads and exports every
symbol include/*.h declares, the registry/errors, and the schedules libmpxa compiles --
simulated on the CPU by tests/plan_sim.py and compared with the oracle."""
import os
import re

import numpy as np
import pytest

import oracle
import synth
from paper_2309_07337_b200 import Plan, list_algorithms, mpxa
from plan_sim import simulate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):        # C-ABI headers only (mpxa_device.cuh is device code)
            continue
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(mpxa_\w+)\s*\(", txt):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_header_symbol():
    lib = mpxa.lib()
    syms = header_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(lib, s), s
    assert syms == set(mpxa.SIGNATURES), "binding signatures must cover exactly the header"


def test_error_strings_and_registry():
    lib = mpxa.lib()
    for s in range(10):
        assert lib.mpxa_error_string(s)
    assert list_algorithms("alltoall") == ["pairwise", "bruck", "hier"]
    assert list_algorithms("alltoallv") == ["pairwise", "hier", "bruck"]
    assert list_algorithms("allgather") == ["pairwise", "bruck", "ring", "hier"]
    assert lib.mpxa_algo_name(2) == b"bruck"


def test_bad_plans_rejected():
    with pytest.raises(mpxa.MpxaError):
        Plan("alltoall", "ring", 4)          # ring is not an alltoall variant
    with pytest.raises(mpxa.MpxaError):
        Plan("alltoall", "hier", 6, g=4)     # p % g != 0


def _topologies(p):
    out = []
    for G in range(1, p + 1):
        if p % G == 0 and G <= 32:
            out.append(G)
    return out


@pytest.mark.parametrize("staged", [0, 1])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 8, 12])
def test_alltoall_plans_simulate_to_oracle(p, staged, monkeypatch):
    """Every variant and GPU split; hierarchical with group = GPU in the fused form (default)
    and the literal three-step form (MPXA_HIER_STAGED=1)."""
    monkeypatch.setenv("MPXA_HIER_STAGED", str(staged))
    b = 3
    send = synth.alltoall_sendbuf(p, p, b)
    want = oracle.alltoall_definition(send)
    for G in _topologies(p):
        for algo in ("pairwise", "bruck"):
            pl = Plan("alltoall", algo, p, G=G)
            got = simulate(pl, send, np.zeros_like(send), b)
            assert np.array_equal(got, want), (algo, G)
        for g in range(1, p + 1):
            if p % g == 0:
                pl = Plan("alltoall", "hier", p, G=G, g=g)
                assert np.array_equal(simulate(pl, send, np.zeros_like(send), b), want), ("hier", G, g)


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 9])
def test_allgather_plans_simulate_to_oracle(p):
    b = 5
    send = synth.allgather_sendbuf(p, p, b)
    want = oracle.allgather_definition(send)
    for G in _topologies(p):
        for algo in ("pairwise", "bruck", "ring"):
            pl = Plan("allgather", algo, p, G=G)
            got = simulate(pl, send, np.zeros((p, p * b), np.uint8), b)
            assert np.array_equal(got, want), (algo, G)


@pytest.mark.parametrize("staged", [0, 1])
@pytest.mark.parametrize("p,g", [(4, 2), (8, 2), (8, 4), (6, 3), (8, 8), (5, 1)])
def test_alltoallv_plans_simulate_to_oracle(p, g, staged, monkeypatch):
    monkeypatch.setenv("MPXA_HIER_STAGED", str(staged))
    for seed in range(4):
        c = synth.cfg4_counts(seed, p, 24)
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed, c, elem=8, packed=bool(seed % 2))
        recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
        want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0)
        for G in _topologies(p):
            for algo, gg in (("pairwise", 1), ("hier", g), ("bruck", 1)):
                pl = Plan("alltoallv", algo, p, G=G, g=gg, counts=sc, sdispls=sd, rdispls=rd)
                got = simulate(pl, send, recv0, 8)
                assert np.array_equal(got, want), (algo, G, seed)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 7, 8, 16])
def test_bruck_stage_plans_match_oracle_intermediate_states(p):
    b = 2
    send = synth.alltoall_sendbuf(7, p, b)
    K = 0
    while (1 << K) < p:
        K += 1
    for stage in range(K + 1):
        _, T, _ = oracle.alltoall(send, "bruck", stop_stage=stage)
        pl = Plan("alltoall", "bruck", p, stop_stage=stage)
        assert np.array_equal(simulate(pl, send, np.zeros_like(send), b), T), stage
        ag = synth.allgather_sendbuf(7, p, b)
        _, Tg, _ = oracle.allgather(ag, "bruck", stop_stage=stage)
        plg = Plan("allgather", "bruck", p, stop_stage=stage)
        got = simulate(plg, ag, np.zeros((p, p * b), np.uint8), b)
        n = min(1 << stage, p) * b
        assert np.array_equal(got[:, :n], Tg[:, :n]), stage


def test_message_counts_of_plans():
    """Inter-GPU messages (signals per launch) against SURVEY.md C.6 / Appendix A."""
    # pairwise over G GPUs, 1 rank each: G(G-1) GPU-pair messages
    assert Plan("alltoall", "pairwise", 8, G=8).info["signals"] == 56
    # Bruck alltoall: K rounds x G messages (one per GPU per round)
    assert Plan("alltoall", "bruck", 8, G=8).info["signals"] == 3 * 8
    # hierarchical, group = GPU (cfg5): exactly G(G-1) inter-GPU messages
    assert Plan("alltoall", "hier", 32, R=4, G=8, g=4).info["signals"] == 56
    # ring allgather: (p-1) steps x G messages
    assert Plan("allgather", "ring", 8, G=8).info["signals"] == 7 * 8
    assert Plan("allgather", "bruck", 8, G=8).info["signals"] == 3 * 8
    # single GPU: no signals at all
    for algo in ("pairwise", "bruck", "hier"):
        assert Plan("alltoall", algo, 8, G=1, g=2).info["signals"] == 0


def test_hier_group_gpu_fused_vs_staged(monkeypatch):
    """Hierarchical with group = GPU: fused = one step, no workspace, the same G(G-1)
    inter-group messages as the staged three-step form."""
    fused = Plan("alltoall", "hier", 32, R=4, G=8, g=4)
    monkeypatch.setenv("MPXA_HIER_STAGED", "1")
    staged = Plan("alltoall", "hier", 32, R=4, G=8, g=4)
    assert fused.info["nsteps"] == 1 and fused.info["work_units"] == 0
    assert staged.info["nsteps"] == 3 and staged.info["work_units"] > 0
    assert fused.info["signals"] == staged.info["signals"] == 8 * 7

"""f1 neighbor alltoallv schedules (libmpxa, host-only plan API) simulated on the CPU and
compared with the oracle (-m "not gpu").

For standard and locality-aware programs on every GPU split, tests/plan_sim.py executes
the moves with the executor's semantics and checks the CTA-ownership properties; the result
must equal oracle.neighbor_definition bit for bit.  The locality program's group-crossing
step must carry exactly the oracle's deduplicated value count."""
import numpy as np
import pytest

import oracle
import synth
from paper_2309_07337_b200 import Plan, MpxaError
from paper_2309_07337_b200 import mpxa as M
from plan_sim import simulate

WORK = 2


def splits(p):
    return [G for G in range(1, p + 1) if p % G == 0 and G <= 32]


def instances():
    yield "ring4", 4, synth.ring_edges(4, 3)
    yield "ring2", 2, synth.ring_edges(2, 2)             # both neighbours are the same rank
    yield "stencil5", 8, synth.stencil_edges(4, 2, 16, 8, corners=False)
    yield "stencil9", 8, synth.stencil_edges(4, 2, 16, 8, corners=True)
    yield "stencil9_16", 16, synth.stencil_edges(4, 4, 16, 16, corners=True)
    for seed in range(6):
        p = [3, 4, 6, 8][seed % 4]
        yield f"random{seed}", p, synth.random_edges(seed, p, 4, 5, 10)
    yield "empty", 4, []


@pytest.mark.parametrize("staged", [0, 1])
@pytest.mark.parametrize("name,p,edges", list(instances()), ids=[x[0] for x in instances()])
def test_neighbor_plans_simulate_to_oracle(name, p, edges, staged, monkeypatch):
    monkeypatch.setenv("MPXA_HIER_STAGED", str(staged))   # group = GPU: fused or three steps
    gr, si, ri = synth.graph_from_edges(p, edges)
    send, recv0 = synth.neighbor_buffers(1, p, gr, si, w=8)
    want = oracle.neighbor_definition(send, recv0, 8, gr)
    for G in splits(p):
        pl = Plan.neighbor(gr, R=p // G, G=G)
        assert np.array_equal(simulate(pl, send, recv0, 8), want), ("standard", G)
        assert pl.info["nsteps"] == (1 if len(edges) and gr["sc"].sum() else 0)
        for g in [x for x in (1, 2, 4, p) if p % x == 0]:
            pl = Plan.neighbor(gr, R=p // G, G=G, g=g, locality=True, send_idx=si, recv_idx=ri)
            got = simulate(pl, send, recv0, 8)
            assert np.array_equal(got, want), ("locality", G, g)


@pytest.mark.parametrize("name,p,edges", [x for x in instances() if x[0] != "empty"],
                         ids=[x[0] for x in instances() if x[0] != "empty"])
def test_locality_crossing_values_match_oracle(name, p, edges):
    """Elements moved between groups in the locality schedule = the oracle's inter-group
    record count = |{(index, src group, dst group)}| (dedup optimality)."""
    gr, si, ri = synth.graph_from_edges(p, edges)
    send, recv0 = synth.neighbor_buffers(2, p, gr, si, w=8)
    for g in [x for x in (1, 2, 4) if p % x == 0]:
        _, st = oracle.neighbor(send, recv0, 8, gr, "locality", g=g, send_idx=si, recv_idx=ri)
        for G in (1, p // g):             # staged (groups inside one GPU) and fused (group = GPU)
            pl = Plan.neighbor(gr, R=p // G, G=G, g=g, locality=True, send_idx=si, recv_idx=ri)
            mv = [m for x in range(G) for m in pl.moves(x)]
            crossing = sum(m.len for m in mv if m.src_rank // g != m.dst_rank // g)
            assert crossing == st["inter_values"], (g, G)


def test_stencil_runs_coalesce():
    """Halo rows / columns travel as runs (one move per boundary segment), not per element."""
    edges = synth.stencil_edges(2, 2, 64, 64, corners=True)
    gr, si, ri = synth.graph_from_edges(4, edges)
    pl = Plan.neighbor(gr, R=1, G=4, g=1, locality=True, send_idx=si, recv_idx=ri)
    n_elem = int(gr["sc"].sum())
    total_moves = pl.info["total_moves"]
    assert total_moves < n_elem // 4


def test_standard_plan_is_one_move_per_edge():
    gr, si, ri = synth.graph_from_edges(8, synth.stencil_edges(4, 2, 16, 8))
    pl = Plan.neighbor(gr, R=2, G=4)
    assert pl.info["total_moves"] == int((gr["sc"] > 0).sum())


def test_neighbor_plan_errors():
    gr, si, ri = synth.graph_from_edges(4, [(0, 2, [7, 8]), (1, 3, [9])])
    bad = dict(gr)
    bad["rc"] = gr["rc"].copy()
    bad["rc"][0] += 1                                           # counts of a pair disagree
    with pytest.raises(MpxaError) as e:
        Plan.neighbor(bad, R=4, G=1)
    assert e.value.status == M.ERR_MISMATCH
    lonely = dict(gr)
    lonely["indeg"] = np.array([0, 0, 0, 1], np.int32)          # an out-edge with no receiver
    lonely["src"], lonely["rc"], lonely["rd"] = gr["src"][1:], gr["rc"][1:], gr["rd"][1:]
    with pytest.raises(MpxaError) as e:
        Plan.neighbor(lonely, R=4, G=1)
    assert e.value.status == M.ERR_MISMATCH
    wrong = ri.copy()
    wrong[0] = 99                                               # received index != sent index
    with pytest.raises(MpxaError) as e:
        Plan.neighbor(gr, R=4, G=1, g=2, locality=True, send_idx=si, recv_idx=wrong)
    assert e.value.status == M.ERR_TOPOLOGY
    with pytest.raises(MpxaError) as e:
        Plan.neighbor(gr, R=4, G=1, g=3, locality=True, send_idx=si, recv_idx=ri)   # 4 % 3
    assert e.value.status == M.ERR_TOPOLOGY


def test_neighbor_registry():
    assert M.list_algorithms("neighbor_alltoallv") == ["pairwise", "locality"]
    assert M.lib().mpxa_algo_name(5) == b"locality"


def test_locality_fused_has_two_steps(monkeypatch):
    """Group = GPU: the gather to the leader is GPU-local and fused into the exchange (two
    steps, no out-aggregates); MPXA_HIER_STAGED=1 keeps the literal three steps."""
    gr, si, ri = synth.graph_from_edges(8, synth.stencil_edges(4, 2, 16, 8, corners=True))
    fused = Plan.neighbor(gr, R=2, G=4, g=2, locality=True, send_idx=si, recv_idx=ri)
    monkeypatch.setenv("MPXA_HIER_STAGED", "1")
    staged = Plan.neighbor(gr, R=2, G=4, g=2, locality=True, send_idx=si, recv_idx=ri)
    assert fused.info["nsteps"] == 2 and staged.info["nsteps"] == 3
    assert fused.info["work_units"] < staged.info["work_units"]

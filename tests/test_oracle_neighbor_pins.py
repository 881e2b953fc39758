"""Pins of the f1 oracle: persistent neighborhood alltoallv, standard and locality-aware
(§2.2).  CPU only (-m "not gpu").

Each pin comes from outside the oracle: MPI's matching rule checked by brute force with a
unique label per (source rank, out-edge, element); the complete graph reducing to the
(already pinned) alltoallv definition; SPEC.md's worked examples (ring message counts,
stencil degree, the "index 7 to ranks 2 and 3" dedup example); closed-form value counts
(standard = elements on group-crossing edges; locality = |{(index, src group, dst group)}|
by enumeration); and the cross-variant equivalence the paper promises ("only needs to be
replaced with the persistent MPIX version").
"""
import numpy as np
import pytest

import oracle
import synth


def labelled_send(p, gr):
    """8-byte element payload = unique label (1 + r, out-edge position k, element x)."""
    ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
    S = max(1, int(max(((gr["sd"] + gr["sc"])[ooff[r]:ooff[r + 1]].max() if ooff[r + 1] > ooff[r] else 0)
                       for r in range(p)))) * 8
    send = np.zeros((p, S), np.uint8)
    for r in range(p):
        for k, e in enumerate(range(ooff[r], ooff[r + 1])):
            for x in range(int(gr["sc"][e])):
                lab = np.array([((1 + r) << 40) | (k << 20) | x], np.uint64).view(np.uint8)
                o = (int(gr["sd"][e]) + x) * 8
                send[r, o:o + 8] = lab
    return send


def recv_size(p, gr):
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])])
    return max(1, int(max(((gr["rd"] + gr["rc"])[ioff[r]:ioff[r + 1]].max() if ioff[r + 1] > ioff[r] else 0)
                          for r in range(p)))) * 8


@pytest.mark.parametrize("seed", range(40))
def test_matching_rule_brute_force(seed):
    """MPI pairs the j-th message r->q with the j-th receive q<-r (multigraph edges)."""
    p = 2 + seed % 4
    edges = synth.random_edges(seed, p, 4, 3, 1000)
    gr, _, _ = synth.graph_from_edges(p, edges)
    send = labelled_send(p, gr)
    recv0 = np.full((p, recv_size(p, gr)), 0xA5, np.uint8)
    got = oracle.neighbor_definition(send, recv0, 8, gr)
    outs = {r: [(d, len(ids)) for (s, d, ids) in edges if s == r] for r in range(p)}
    expect = recv0.copy()
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])])
    for q in range(p):
        seen = {}
        for e in range(ioff[q], ioff[q + 1]):
            r = int(gr["src"][e])
            j = seen.get(r, 0)
            seen[r] = j + 1
            ks = [k for k, (d, _) in enumerate(outs[r]) if d == q]
            k = ks[j]
            for x in range(int(gr["rc"][e])):
                lab = np.array([((1 + r) << 40) | (k << 20) | x], np.uint64).view(np.uint8)
                o = (int(gr["rd"][e]) + x) * 8
                expect[q, o:o + 8] = lab
    assert np.array_equal(got, expect)
    r2, st = oracle.neighbor(send, recv0, 8, gr, "standard")
    assert np.array_equal(r2, expect)
    assert st["msgs"] == int((gr["sc"] > 0).sum())           # one message per non-empty edge


def test_complete_graph_is_alltoallv():
    p = 5
    rng = np.random.default_rng(3)
    counts = rng.integers(0, 4, size=(p, p))
    edges = [(r, j, list(range(int(counts[r, j])))) for r in range(p) for j in range(p)]
    gr, _, _ = synth.graph_from_edges(p, edges)
    send = rng.integers(0, 256, size=(p, 8 * int(counts.sum(1).max() + 1)), dtype=np.uint8)
    recv0 = np.zeros((p, 8 * int(counts.sum(0).max() + 1)), np.uint8)
    sc = counts.astype(np.int64)
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
    rc = sc.T.copy()
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0)
    assert np.array_equal(oracle.neighbor_definition(send, recv0, 8, gr), want)


def test_spec_ring_example():
    """ring topology, 4 ranks, count 1 -> each start sends exactly 2 messages per
    rank; rank q's edge from q-1 holds what q-1 sent to q (and likewise from q+1)."""
    p = 4
    gr, si, ri = synth.graph_from_edges(p, synth.ring_edges(p, 1))
    send = labelled_send(p, gr)
    recv, st = oracle.neighbor(send, np.zeros((p, 16), np.uint8), 8, gr, "standard")
    assert st["msgs"] == 8 and st["max_msgs_per_rank"] == 2
    ioff = np.concatenate([[0], np.cumsum(gr["indeg"])])
    for q in range(p):
        assert sorted(int(r) for r in gr["src"][ioff[q]:ioff[q + 1]]) == sorted(((q - 1) % p, (q + 1) % p))
        for slot, e in enumerate(range(ioff[q], ioff[q + 1])):
            r = int(gr["src"][e])
            k = 0 if q == (r - 1) % p else 1                      # r's out-edges: r-1 first, then r+1
            lab = np.array([((1 + r) << 40) | (k << 20)], np.uint64).view(np.uint8)
            assert np.array_equal(recv[q, 8 * slot:8 * slot + 8], lab)


def test_spec_stencil_degree():
    """5-point stencil on a 4x4 rank grid -> per-rank messages = its degree."""
    edges = synth.stencil_edges(4, 4, 16, 16, corners=False)
    gr, si, ri = synth.graph_from_edges(16, edges)
    send, recv0 = synth.neighbor_buffers(0, 16, gr, si)
    _, st = oracle.neighbor(send, recv0, 8, gr, "standard")
    deg = gr["outdeg"]
    assert st["msgs"] == int(deg.sum()) and st["max_msgs_per_rank"] == int(deg.max()) == 4
    assert sorted(set(int(d) for d in deg)) == [2, 3, 4]        # corners, edges, interior


def test_spec_dedup_example():
    """rank 0 (node 0) sends global index 7 to ranks 2 and 3 (both node 1):
    standard -> 2 inter-node values; locality-aware -> 1."""
    p, g = 4, 2
    gr, si, ri = synth.graph_from_edges(p, [(0, 2, [7]), (0, 3, [7])])
    send, recv0 = synth.neighbor_buffers(5, p, gr, si)
    want = oracle.neighbor_definition(send, recv0, 8, gr)
    rs, st_s = oracle.neighbor(send, recv0, 8, gr, "standard", ppn=g)
    rl, st_l = oracle.neighbor(send, recv0, 8, gr, "locality", g=g, send_idx=si, recv_idx=ri)
    assert st_s["inter_bytes"] == 2 * 8
    assert st_l["inter_values"] == 1
    assert np.array_equal(rs, want) and np.array_equal(rl, want)


def crossing_counts(gr, si, g, p):
    ooff = np.concatenate([[0], np.cumsum(gr["outdeg"])])
    std, triples, e0 = 0, set(), 0
    for r in range(p):
        for e in range(ooff[r], ooff[r + 1]):
            n = int(gr["sc"][e])
            d = int(gr["dst"][e])
            if r // g != d // g:
                std += n
                for x in si[e0:e0 + n]:
                    triples.add((int(x), r // g, d // g))
            e0 += n
    return std, len(triples)


@pytest.mark.parametrize("seed", range(30))
def test_locality_equivalence_and_dedup_optimality(seed):
    """Variant equivalence and dedup optimality: records crossing groups =
    |{(index, src group, dst group)}| by enumeration; <= the standard element count."""
    p = [2, 4, 6, 8][seed % 4]
    g = [1, 2, 2, 4, 3][seed % 5] if p % [1, 2, 2, 4, 3][seed % 5] == 0 else 2
    edges = synth.random_edges(seed, p, 4, 6, 12)            # small id space: many duplicates
    gr, si, ri = synth.graph_from_edges(p, edges)
    send, recv0 = synth.neighbor_buffers(seed, p, gr, si)
    want = oracle.neighbor_definition(send, recv0, 8, gr)
    rl, st = oracle.neighbor(send, recv0, 8, gr, "locality", g=g, send_idx=si, recv_idx=ri)
    assert np.array_equal(rl, want)
    std, uniq = crossing_counts(gr, si, g, p)
    assert st["inter_values"] == uniq <= std


def test_locality_without_duplicates_equals_standard_count():
    """no duplicate indices -> inter-group values equal the standard variant's."""
    edges = synth.stencil_edges(4, 2, 32, 16, corners=False)
    n = 0
    uniq_edges = []
    for s_, d_, ids in edges:                                   # re-label: every element unique
        uniq_edges.append((s_, d_, list(range(n, n + len(ids)))))
        n += len(ids)
    gr, si, ri = synth.graph_from_edges(8, uniq_edges)
    send, recv0 = synth.neighbor_buffers(2, 8, gr, si)
    want = oracle.neighbor_definition(send, recv0, 8, gr)
    for g in (1, 2, 4):
        std, uniq = crossing_counts(gr, si, g, 8)
        r, st = oracle.neighbor(send, recv0, 8, gr, "locality", g=g, send_idx=si, recv_idx=ri)
        assert st["inter_values"] == std == uniq
        assert np.array_equal(r, want)


def test_stencil_corners_dedup():
    """9-point halo with 2 ranks per group: a corner point bound for two ranks of one remote
    group crosses once."""
    edges = synth.stencil_edges(4, 2, 32, 16, corners=True)
    gr, si, ri = synth.graph_from_edges(8, edges)
    send, recv0 = synth.neighbor_buffers(3, 8, gr, si)
    want = oracle.neighbor_definition(send, recv0, 8, gr)
    std, uniq = crossing_counts(gr, si, 2, 8)
    rl, st = oracle.neighbor(send, recv0, 8, gr, "locality", g=2, send_idx=si, recv_idx=ri)
    assert np.array_equal(rl, want)
    assert st["inter_values"] == uniq < std


def test_inconsistent_recv_indices_rejected():
    gr, si, ri = synth.graph_from_edges(4, [(0, 2, [7, 8]), (1, 3, [9])])
    send, recv0 = synth.neighbor_buffers(0, 4, gr, si)
    bad = ri.copy()
    bad[0] = 99
    with pytest.raises(ValueError):
        oracle.neighbor(send, recv0, 8, gr, "locality", g=2, send_idx=si, recv_idx=bad)


def test_empty_topology():
    """empty topology -> zero messages, recv untouched."""
    gr, si, ri = synth.graph_from_edges(3, [])
    send = np.zeros((3, 8), np.uint8)
    recv0 = np.full((3, 8), 0xA5, np.uint8)
    for variant in ("standard", "locality"):
        r, st = oracle.neighbor(send, recv0, 8, gr, variant, g=1, send_idx=si, recv_idx=ri)
        assert st["msgs"] == 0 and np.array_equal(r, recv0)


def test_mutations_fail_a_pin():
    """A wrong matching rule (first edge always) or a dropped dedup would break the pins
    above; check the pins can tell: swapping two multigraph edges changes the result."""
    gr, si, ri = synth.graph_from_edges(2, [(0, 1, [1]), (0, 1, [2])])
    send = labelled_send(2, gr)
    recv = oracle.neighbor_definition(send, np.zeros((2, 16), np.uint8), 8, gr)
    first = np.array([(1 << 40) | (0 << 20)], np.uint64).view(np.uint8)
    second = np.array([(1 << 40) | (1 << 20)], np.uint64).view(np.uint8)
    assert np.array_equal(recv[1, :8], first) and np.array_equal(recv[1, 8:], second)
    assert not np.array_equal(first, second)

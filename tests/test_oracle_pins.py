"""Pins for the CPU oracle, run with -m "not gpu".

Each check compares the oracle against something other than itself: numpy transposes
and concatenations (library routines), brute force with unique byte labels, closed-form
message counts, the Bruck per-round invariants, and hand-written golden fixtures
(tests/golden/spec_examples.json, each entry citing PAPER.md / SPEC.md).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
VARIANTS_A2A = ["pairwise", "bruck"]


def ceil_log2(p):
    k = 0
    while (1 << k) < p:
        k += 1
    return k


def labelled_alltoall_send(p, b):
    """Byte k of block (src -> dst) = unique label src*25*... (p <= 5, b <= 3 -> < 256)."""
    s = np.zeros((p, p * b), dtype=np.uint8)
    for src in range(p):
        for dst in range(p):
            for k in range(b):
                s[src, dst * b + k] = (src * 5 + dst) * 3 + k + 1   # 1..75, never 0
    return s


def check_labels_alltoall(recv, p, b):
    for r in range(p):
        for j in range(p):
            for k in range(b):
                lab = int(recv[r, j * b + k]) - 1
                src, rem = divmod(lab // 3, 5)
                assert (src, rem, lab % 3) == (j, r, k), (r, j, k, lab)


# ---------------------------------------------------------------- definitions vs numpy

@pytest.mark.parametrize("p,b", [(1, 5), (2, 1), (3, 7), (4, 16), (7, 3), (8, 64), (16, 4)])
def test_alltoall_definition_is_block_transpose(p, b):
    send = synth.alltoall_sendbuf(p * 100 + b, p, b)
    ref = send.reshape(p, p, b).transpose(1, 0, 2).reshape(p, p * b)   # numpy, textbook
    assert np.array_equal(oracle.alltoall_definition(send), ref)


@pytest.mark.parametrize("p,b", [(1, 3), (2, 1), (5, 9), (8, 32)])
def test_allgather_definition_is_concatenation(p, b):
    send = synth.allgather_sendbuf(7, p, b)
    cat = np.concatenate(list(send))
    assert np.array_equal(oracle.allgather_definition(send), np.tile(cat, (p, 1)))
    for T in (1, 2, 3, 8):       # the row-split (host-threaded) form: the same concatenation
        assert np.array_equal(oracle.allgather_definition_threaded(send, T), np.tile(cat, (p, 1))), T


# ---------------------------------------------------------------- brute force, labels

@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("b", [0, 1, 2, 3])
def test_alltoall_bruteforce_labels_all_variants(p, b):
    send = labelled_alltoall_send(p, b)
    outs = [oracle.alltoall_definition(send)]
    for v in VARIANTS_A2A:
        outs.append(oracle.alltoall(send, v)[0])
    for g in range(1, p + 1):
        if p % g == 0:
            outs.append(oracle.alltoall(send, "hier", g=g)[0])
    for o in outs:
        check_labels_alltoall(o, p, b)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("b", [0, 1, 2, 3])
def test_allgather_bruteforce_labels_all_variants(p, b):
    send = np.zeros((p, b), dtype=np.uint8)
    for r in range(p):
        for k in range(b):
            send[r, k] = r * 3 + k + 1
    for out in [oracle.allgather_definition(send)] + [oracle.allgather(send, v)[0] for v in ("bruck", "ring", "direct")]:
        for r in range(p):
            for j in range(p):
                for k in range(b):
                    assert int(out[r, j * b + k]) - 1 == j * 3 + k


def _v_instance_from_counts(c, w=1, canary=0xA5):
    """Labelled alltoallv instance: byte k of segment (src->dst) = src*16 + dst*4 + k (p<=3, count<=2, w=1)."""
    p = c.shape[0]
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c, elem=w, packed=True)
    for src in range(p):
        for dst in range(p):
            for k in range(int(c[src, dst]) * w):
                send[src, sd[src, dst] * w + k] = src * 16 + dst * 4 + k
    recv0 = np.full((p, Rcap), canary, dtype=np.uint8)
    return send, sc, sd, rc, rd, recv0


def _check_v_labels(out, c, rd, w=1, canary=0xA5):
    p = c.shape[0]
    expected = np.full_like(out, canary)
    for r in range(p):
        for j in range(p):
            for k in range(int(c[j, r]) * w):
                expected[r, rd[r, j] * w + k] = j * 16 + r * 4 + k
    assert np.array_equal(out, expected)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_alltoallv_every_count_matrix_0_to_2(p):
    """Every count matrix with entries in {0,1,2} (p <= 3: 1, 16... 19683 instances)."""
    variants = [("pairwise", 0), ("bruck", 0)] + [("hier", g) for g in range(1, p + 1) if p % g == 0]
    for flat in itertools.product(range(3), repeat=p * p):
        c = np.array(flat, dtype=np.int64).reshape(p, p)
        send, sc, sd, rc, rd, recv0 = _v_instance_from_counts(c)
        _check_v_labels(oracle.alltoallv_definition(send, sc, sd, rc, rd, 1, recv0), c, rd)
        if p == 3 and sum(flat) % 7:   # full variant sweep on a 1/7-ish subset at p=3 (runtime)
            continue
        for v, g in variants:
            out, st = oracle.alltoallv(send, sc, sd, rc, rd, 1, recv0, variant=v, g=g)
            _check_v_labels(out, c, rd)


@pytest.mark.parametrize("p", [4, 5, 8, 16])
def test_alltoallv_seeded_instances_int64_labels(p):
    """Seeded instances (SPEC.md:552 AC1 idea), int64 elements labelled (src, dst, k)."""
    rng_seeds = range(40 if p <= 8 else 10)
    for seed in rng_seeds:
        c = synth.cfg4_counts(seed, p, 64)            # counts in elements, 10% zeros
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed, c, elem=8, packed=bool(seed % 2))
        s64 = send.view(np.int64)
        for a in range(p):
            for b in range(p):
                for k in range(int(c[a, b])):
                    s64[a, sd[a, b] + k] = (a << 40) | (b << 20) | k
        recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
        outs = [oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0)]
        outs.append(oracle.alltoallv(send, sc, sd, rc, rd, 8, recv0, "pairwise")[0])
        outs.append(oracle.alltoallv(send, sc, sd, rc, rd, 8, recv0, "bruck")[0])
        for g in (2, 4):
            if p % g == 0:
                outs.append(oracle.alltoallv(send, sc, sd, rc, rd, 8, recv0, "hier", g=g)[0])
        covered = np.zeros((p, Rcap), dtype=bool)
        for r in range(p):
            for j in range(p):
                o = rd[r, j] * 8
                covered[r, o:o + c[j, r] * 8] = True
        for out in outs:
            o64 = out.view(np.uint8)
            assert np.all(o64[~covered] == 0xA5)
            for r in range(p):
                for j in range(p):
                    seg = out[r, rd[r, j] * 8:(rd[r, j] + c[j, r]) * 8].view(np.int64)
                    want = (j << 40) | (r << 20) | np.arange(int(c[j, r]), dtype=np.int64)
                    assert np.array_equal(seg, want)


# ---------------------------------------------------------------- variant equivalence

@pytest.mark.parametrize("p", list(range(1, 17)))
def test_alltoall_variants_equal_definition(p):
    for b in (1, 4, 12):
        send = synth.alltoall_sendbuf(1000 + p, p, b)
        ref = send.reshape(p, p, b).transpose(1, 0, 2).reshape(p, p * b)
        for v in VARIANTS_A2A:
            assert np.array_equal(oracle.alltoall(send, v)[0], ref), v
        for g in range(1, p + 1):
            if p % g == 0:
                assert np.array_equal(oracle.alltoall(send, "hier", g=g)[0], ref), g


@pytest.mark.parametrize("p", list(range(1, 17)))
def test_allgather_variants_equal_concatenation(p):
    send = synth.allgather_sendbuf(p, p, 6)
    ref = np.tile(np.concatenate(list(send)), (p, 1))
    for v in ("bruck", "ring", "direct"):
        assert np.array_equal(oracle.allgather(send, v)[0], ref), v


# ---------------------------------------------------------------- Bruck intermediate states

def m_k(p, k):
    """Closed form for |{i < p : bit k of i is 1}| (SURVEY.md §8 notation)."""
    return (p // 2 ** (k + 1)) * 2 ** k + max(0, p % 2 ** (k + 1) - 2 ** k)


@pytest.mark.parametrize("p", list(range(1, 17)) + [32])
def test_bruck_alltoall_round_invariant(p):
    """After round k, T_r[i] holds the block sent by s = (r - (i mod 2^(k+1))) mod p to
    (s + i) mod p; after the rotation (k = -1) s = r."""
    b = 2
    send = synth.alltoall_sendbuf(p, p, b)
    blocks = send.reshape(p, p, b)
    for stage in range(0, ceil_log2(p) + 1):
        k = stage - 1
        _, T, _ = oracle.alltoall(send, "bruck", stop_stage=stage)
        T = T.reshape(p, p, b)
        for r in range(p):
            for i in range(p):
                s = (r - (i % (2 ** (k + 1)))) % p
                assert np.array_equal(T[r, i], blocks[s, (s + i) % p]), (stage, r, i)


@pytest.mark.parametrize("p", list(range(1, 17)))
def test_bruck_allgather_round_invariant(p):
    """After round k, T_r[i] = send_{(r+i) mod p} for i < min(2^(k+1), p) (C.4 item 3)."""
    send = synth.allgather_sendbuf(3, p, 5)
    for stage in range(0, ceil_log2(p) + 1):
        _, T, _ = oracle.allgather(send, "bruck", stop_stage=stage)
        T = T.reshape(p, p, 5)
        for r in range(p):
            for i in range(min(2 ** stage, p)):
                assert np.array_equal(T[r, i], send[(r + i) % p])


# ---------------------------------------------------------------- closed-form counters

@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8, 16])
def test_message_count_closed_forms(p):
    b = 3
    send = synth.alltoall_sendbuf(5, p, b)
    K = ceil_log2(p)
    st = oracle.alltoall(send, "pairwise")[2]
    assert st["msgs"] == p * p and st["bytes"] == p * p * b
    st = oracle.alltoall(send, "bruck")[2]
    assert st["msgs"] == p * K and st["rounds"] == K
    assert st["bytes"] == p * b * sum(m_k(p, k) for k in range(K))
    ag = synth.allgather_sendbuf(5, p, b)
    st = oracle.allgather(ag, "bruck")[2]
    assert st["msgs"] == p * K and st["bytes"] == p * (p - 1) * b
    st = oracle.allgather(ag, "ring")[2]
    assert st["msgs"] == p * (p - 1) and st["max_msgs_per_rank"] == p - 1
    st = oracle.allgather(ag, "direct")[2]
    assert st["msgs"] == p * (p - 1)
    for g in range(1, p + 1):
        if p % g == 0:
            G = p // g
            st = oracle.alltoall(send, "hier", g=g)[2]
            assert st["inter_msgs"] == G * (G - 1)
            # hierarchical never increases inter-node messages vs pairwise
            pw = oracle.alltoall(send, "pairwise", ppn=g)[2]
            assert st["inter_msgs"] <= pw["inter_msgs"]
            assert pw["inter_msgs"] == p * p - G * g * g


def test_golden_message_counts():
    gm = GOLD["message_counts"]
    send = synth.alltoall_sendbuf(1, 4, 2)
    assert oracle.alltoall(send, "pairwise")[2]["msgs"] == gm["pairwise_p4_total_msgs"]
    send16 = synth.alltoall_sendbuf(1, 16, 2)
    assert oracle.alltoall(send16, "hier", g=4)[2]["inter_msgs"] == gm["hier_4nodes_x4_inter_msgs"]
    st = oracle.allgather(synth.allgather_sendbuf(1, 5, 2), "bruck")[2]
    assert st["max_msgs_per_rank"] == gm["bruck_allgather_p5_msgs_per_rank"]
    for key, per_round in GOLD["bruck_alltoall_blocks_per_round"].items():
        if not key.startswith("p"):
            continue
        p = int(key[1:])
        assert [m_k(p, k) for k in range(ceil_log2(p))] == per_round
        send = synth.alltoall_sendbuf(1, p, 1)
        assert oracle.alltoall(send, "bruck")[2]["bytes"] == p * sum(per_round)


# ---------------------------------------------------------------- golden fixtures

def _enc(rows):
    return np.array([[ord(ch) for ch in "".join(r)] for r in rows], dtype=np.uint8)


def test_golden_alltoall_p3():
    g = GOLD["alltoall_p3_labels"]
    send = _enc(g["send"])
    want = _enc(g["recv"])
    assert np.array_equal(oracle.alltoall_definition(send), want)
    for v in VARIANTS_A2A:
        assert np.array_equal(oracle.alltoall(send, v)[0], want)
    assert np.array_equal(oracle.alltoall(send, "hier", g=3)[0], want)


def test_golden_allgather_p3():
    g = GOLD["allgather_p3_labels"]
    send = _enc([[s] for s in g["send"]])
    want = _enc(g["recv"])
    for v in ("bruck", "ring", "direct"):
        assert np.array_equal(oracle.allgather(send, v)[0], want)


def test_golden_alltoallv_p2():
    g = GOLD["alltoallv_p2_labels"]
    send = _enc([[s] for s in g["sendbuf"]])
    recv0 = np.full((2, g["recv_capacity"]), ord(g["canary"]), dtype=np.uint8)
    want = _enc([[s] for s in g["recv"]])
    args = [np.array(g[k], dtype=np.int64) for k in ("sendcounts", "sdispls", "recvcounts", "rdispls")]
    assert np.array_equal(oracle.alltoallv_definition(send, *args, 1, recv0), want)
    for v, gg in (("pairwise", 0), ("hier", 1), ("hier", 2)):
        assert np.array_equal(oracle.alltoallv(send, *args, 1, recv0, v, g=gg)[0], want)


# ---------------------------------------------------------------- special cases

def test_p1_identity_and_zero_counts():
    send = synth.alltoall_sendbuf(9, 1, 13)
    for v in VARIANTS_A2A:
        assert np.array_equal(oracle.alltoall(send, v)[0], send)
    c = np.zeros((4, 4), dtype=np.int64)
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c)
    recv0 = np.full((4, Rcap), 0x5A, dtype=np.uint8)
    for v, g in (("pairwise", 0), ("hier", 2)):
        out, st = oracle.alltoallv(send, sc, sd, rc, rd, 8, recv0, v, g=g)
        assert np.array_equal(out, recv0)
        assert st["bytes"] == 0


def test_counts_exchange_matches_numpy():
    for p in (1, 3, 8, 32):
        sc = synth.cfg4_counts(p, p, 4096)
        rc, rd, st = oracle.counts_exchange(sc)
        assert np.array_equal(rc, sc.T)                                  # transpose identity
        assert np.array_equal(rd[:, 1:], np.cumsum(rc, axis=1)[:, :-1])  # exclusive scan
        assert np.all(rd[:, 0] == 0)
        assert st["msgs"] == p * p


def test_bad_arguments_rejected():
    c = np.ones((2, 2), dtype=np.int64)
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c)
    recv0 = np.zeros((2, Rcap), dtype=np.uint8)
    bad = sc.copy()
    bad[0, 1] = 2          # sendcounts[0->1] != recvcounts[1<-0]
    with pytest.raises(RuntimeError):
        oracle.alltoallv(send, bad, sd, rc, rd, 8, recv0)
    with pytest.raises(RuntimeError):
        oracle.alltoallv(send, sc, sd, rc, rd, 8, recv0, "hier", g=3)   # p % g != 0


# ---- f2(i): hierarchical allgather ----------------------------------------

@pytest.mark.parametrize("p,g", [(1, 1), (4, 2), (8, 2), (8, 4), (6, 3), (16, 4), (12, 4), (5, 5), (6, 1)])
def test_allgather_hier_concatenation_and_counts(p, g):
    """Equals numpy concatenation; inter-node messages = G * ceil(log2 G) (Bruck among the G
    leaders, SPEC.md:236's count per rank) -- every other message stays inside a node."""
    send = synth.allgather_sendbuf(p, p, 7)
    recv, _, st = oracle.allgather(send, "hier", g=g)
    assert np.array_equal(recv, np.tile(send.reshape(1, -1), (p, 1)))
    G = p // g
    K = 0 if G == 1 else int(np.ceil(np.log2(G)))
    assert st["inter_msgs"] == G * K
    assert st["intra_msgs"] == p + p                 # gather (incl. leader loopback) + broadcast


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 13])
def test_alltoallv_bruck_message_counts(p):
    """Bruck-v keeps Bruck's message count: ceil(log2 p) messages per rank."""
    c = synth.cfg4_counts(p, p, 40)
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(p, c, elem=8)
    out, st = oracle.alltoallv(send, sc, sd, rc, rd, 8, np.zeros((p, Rcap), np.uint8), "bruck")
    K = 0 if p == 1 else int(np.ceil(np.log2(p)))
    assert st["msgs"] == p * K and st["max_msgs_per_rank"] == K
    assert np.array_equal(out, oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, np.zeros((p, Rcap), np.uint8)))

"""GPU parity: libmpxa (C ABI, sm_100a kernels) vs the CPU oracle, bit-exact (-m gpu).

Inputs come from synth/ (seeded); expected values from oracle/ only.  Payloads are opaque
bytes, so the bar is bit-exactness for every op, variant, size and topology, including
ragged / misaligned sizes, zero counts, canaries outside received ranges, emulated
multi-GPU protocol runs, Bruck intermediate states and persistent start/wait cycles.
"""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2309_07337_b200 import Comm, MpxaError  # noqa: E402
from paper_2309_07337_b200 import mpxa as M  # noqa: E402

DEV = "cuda:0"
_COMMS = {}


def comm(p, G=0, g=0):
    key = (p, G, g)
    if key not in _COMMS:
        _COMMS[key] = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=g, timeout_s=20.0)
    return _COMMS[key]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def topologies(p):
    return [G for G in (0, 2, 4, 8) if G == 0 or (p % G == 0 and G <= p)]


def run_alltoall(c, send, algo):
    d_send = dev(send)
    d_recv = torch.full_like(d_send, 0xA5)
    c.alltoall(d_send, d_recv, algo=algo, count=send.shape[1] // c.p)
    out = host(d_recv)
    assert c.check() == 0
    return out


# ------------------------------------------------------------------ cfg1 (configs[0])

@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("algo", ["pairwise", "bruck", "hier"])
def test_cfg1_alltoall_p4_8xint32(seed, algo):
    p = 4
    send = np.stack([np.concatenate([synth.cfg1_block(seed, r, j) for j in range(p)]) for r in range(p)])
    send8 = send.view(np.uint8)
    want = oracle.alltoall_definition(send8)
    for G in (0, 2, 4):
        for g in (2, 4):
            c = comm(p, G, g)
            d_send = dev(send)               # int32 words, count = 8 per destination
            d_recv = torch.zeros_like(d_send)
            c.alltoall(d_send, d_recv, algo=algo)
            assert np.array_equal(host(d_recv).view(np.uint8), want), (G, g)


# ------------------------------------------------------------------ alltoall sweeps

SIZES = [1, 3, 4, 8, 16, 48, 100, 1000, 4096 + 12, 65536 + 128, 300_000]


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 7, 8, 16])
def test_alltoall_all_variants_sizes(p):
    for b in SIZES:
        if p * p * b > 64 << 20:
            continue
        send = synth.alltoall_sendbuf(b + p, p, b)
        want = oracle.alltoall_definition(send)
        for G in topologies(p):
            for algo in ("pairwise", "bruck", "hier"):
                g = 2 if p % 2 == 0 else 1
                got = run_alltoall(comm(p, G, g), send, algo)
                assert np.array_equal(got, want), (p, b, G, algo)


@pytest.mark.parametrize("p,g", [(8, 2), (8, 4), (6, 3), (4, 4), (8, 8), (32, 4)])
def test_alltoall_hier_groups(p, g):
    b = 260
    send = synth.alltoall_sendbuf(11, p, b)
    want = oracle.alltoall_definition(send)
    for G in topologies(p) + ([] if p != 32 else [32 // 4]):
        got = run_alltoall(comm(p, G, g), send, "hier")
        assert np.array_equal(got, want), (G,)


def test_cfg3_float32_payload_opaque_nan():
    """cfg3 float32 U[-1,1) blocks + NaN/denormal bit patterns survive bit-exactly."""
    p, count = 8, 1024 + 3
    send = np.stack([np.concatenate([synth.cfg3_block(5, r, j, count) for j in range(p)]) for r in range(p)])
    raw = send.view(np.uint32)
    raw[:, ::97] = 0x7FC00001      # quiet NaN with payload
    raw[:, 1::89] = 0x00000001     # denormal
    raw[:, 2::83] = 0xFF800000     # -inf
    want = oracle.alltoall_definition(send.view(np.uint8))
    for algo in ("pairwise", "bruck", "hier"):
        for G in (0, 8):
            c = comm(p, G, 2)
            d_send = dev(send)
            d_recv = torch.zeros_like(d_send)
            c.alltoall(d_send, d_recv, algo=algo)
            assert np.array_equal(host(d_recv).view(np.uint8), want), (algo, G)


def test_cfg5_bf16_payload_p32():
    """cfg5 shape on one device: p=32 ranks, bf16 N(0,1) payload, 4 ranks per (virtual) GPU."""
    p, count = 32, 8 + 64
    send = np.stack([np.concatenate([synth.cfg5_block(3, r, j, count) for j in range(p)]) for r in range(p)])
    want = oracle.alltoall_definition(send.view(np.uint8))
    for algo in ("pairwise", "bruck", "hier"):
        for G in (0, 8):
            c = comm(p, G, 4)
            d_send = dev(send).view(torch.bfloat16)
            d_recv = torch.zeros_like(d_send)
            c.alltoall(d_send, d_recv, algo=algo)
            assert np.array_equal(host(d_recv.view(torch.int16)).view(np.uint8), want), (algo, G)


def test_misaligned_pointers():
    """recv / send at odd byte offsets exercise the 8/4/2/1-byte copy paths."""
    p, b = 4, 777
    send = synth.alltoall_sendbuf(3, p, b)
    want = oracle.alltoall_definition(send)
    c = comm(p)
    for so, ro in ((1, 0), (0, 3), (5, 7), (8, 4), (2, 6)):
        bs = torch.zeros(p * p * b + 64, dtype=torch.uint8, device=DEV)
        br = torch.zeros(p * p * b + 64, dtype=torch.uint8, device=DEV)
        bs[so:so + p * p * b] = dev(send.reshape(-1))
        for algo in ("pairwise", "bruck", "hier"):
            br.fill_(0)
            c.alltoall(bs[so:so + p * p * b], br[ro:ro + p * p * b], algo=algo, count=b)
            got = host(br)[ro:ro + p * p * b].reshape(p, p * b)
            assert np.array_equal(got, want), (so, ro, algo)


def test_zero_count_is_noop():
    c = comm(4)
    d = torch.empty(0, dtype=torch.uint8, device=DEV)
    r = torch.full((16,), 7, dtype=torch.uint8, device=DEV)
    c.alltoall(d, r, count=0)
    c.allgather(d, r, count=0)
    assert np.all(host(r) == 7)


# ------------------------------------------------------------------ allgather (cfg2 shape)

@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 16])
def test_allgather_all_variants(p):
    for b in [1, 4, 7, 64, 1000, 4096, 65536 + 5, 1 << 20]:
        if p * p * b > 64 << 20:
            continue
        send = synth.allgather_sendbuf(b, p, b)
        want = oracle.allgather_definition(send)
        for G in topologies(p):
            c = comm(p, G)
            for algo in ("pairwise", "bruck", "ring", "hier"):
                d_send = dev(send)
                d_recv = torch.full((p, p * b), 0x5A, dtype=torch.uint8, device=DEV)
                c.allgather(d_send, d_recv, algo=algo)
                assert np.array_equal(host(d_recv), want), (p, b, G, algo)
            if p % 2 == 0 and b in (7, 4096, 1 << 20):          # locality-aware groups of 2 ranks
                c2 = comm(p, G, 2)
                d_recv = torch.full((p, p * b), 0x5A, dtype=torch.uint8, device=DEV)
                c2.allgather(dev(send), d_recv, algo="hier")
                assert np.array_equal(host(d_recv), want), (p, b, G, "hier g=2")


# ------------------------------------------------------------------ Bruck intermediate states

@pytest.mark.parametrize("p", [2, 3, 4, 5, 8, 16])
def test_bruck_intermediate_states(p):
    b = 36
    send = synth.alltoall_sendbuf(p, p, b)
    ag = synth.allgather_sendbuf(p, p, b)
    K = max(0, int(np.ceil(np.log2(p))))
    for G in topologies(p):
        c = comm(p, G)
        for stage in range(K + 1):
            _, T, _ = oracle.alltoall(send, "bruck", stop_stage=stage)
            d_T = torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
            c.alltoall_bruck_stage(dev(send), d_T, stage)
            assert np.array_equal(host(d_T), T), ("alltoall", G, stage)
            _, Tg, _ = oracle.allgather(ag, "bruck", stop_stage=stage)
            d_Tg = torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
            c.allgather_bruck_stage(dev(ag), d_Tg, stage)
            n = min(1 << stage, p) * b
            assert np.array_equal(host(d_Tg)[:, :n], Tg[:, :n]), ("allgather", G, stage)


# ------------------------------------------------------------------ alltoallv (cfg4 shape)

@pytest.mark.parametrize("mean", [64, 4096, 65536])
@pytest.mark.parametrize("packed", [True, False])
def test_cfg4_alltoallv(mean, packed):
    p = 8
    for seed in (0, 1, 2):
        c4 = synth.cfg4_counts(seed, p, mean)
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed, c4, elem=8, packed=packed)
        recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
        want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0)
        for G in (0, 2, 8):
            for algo, g in (("pairwise", 2), ("hier", 2), ("hier", 4), ("bruck", 2)):
                c = comm(p, G, g)
                d_send = dev(send.view(np.int64))
                d_recv = dev(recv0.view(np.int64))
                c.alltoallv(d_send, sc, sd, d_recv, rc, rd, algo=algo)
                assert np.array_equal(host(d_recv).view(np.uint8), want), (seed, G, algo, g)


@pytest.mark.parametrize("elem", [8, 4])
@pytest.mark.parametrize("packed", [True, False])
def test_cfg4_alltoallv_mean_4MiB(elem, packed, monkeypatch):
    """cfg4 at its real mean (4 MiB per pair, p = 8, 10 % zero pairs): the dynamic work-queue
    executor in warp-ring mode: every warp streams its pieces through its own TMA ring, and
    segments that are only 8-B (int64) or 4-B (int32) congruent are stored 16 B at a time,
    shifted out of shared memory.  Bit-exact with the oracle's slice identity, canaries
    outside the segments untouched; also with MPXA_NO_WRING=1 (the LSU-register queue) and
    over 2 emulated GPUs."""
    p = 8
    for seed in (0, 1):
        c4 = synth.cfg4_counts(seed, p, 4 << 20, elem=elem)
        send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed, c4, elem=elem, packed=packed)
        recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
        want = oracle.alltoallv_definition(send, sc, sd, rc, rd, elem, recv0)
        d_send = dev(send)
        for G, wring in ((0, True), (0, False), (2, True)):
            if wring:
                monkeypatch.delenv("MPXA_NO_WRING", raising=False)
            else:
                monkeypatch.setenv("MPXA_NO_WRING", "1")
            c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, timeout_s=20.0)
            d_recv = dev(recv0)
            c.alltoallv(d_send, sc, sd, d_recv, rc, rd, algo="pairwise", dtype_size=elem)
            path = c.last_launch_path()
            assert np.array_equal(host(d_recv), want), (seed, G, wring)
            if G == 0 and os.environ.get("MPXA_NO_DYN", "0") == "0":   # (path knobs off)
                assert "dyn" in path and (("wring" in path) == wring), path
            c.finalize()


@pytest.mark.parametrize("dyn", [True, False, "wring"])
def test_alltoallv_large_misaligned(dyn, monkeypatch):
    """Large byte-granular alltoallv (dtype 1, 0.5-1.5 MiB per pair, 0-15 byte gaps between
    segments): every source/destination misalignment class, through the dynamic work-queue
    executor (TMA queue for 16-B congruent segments, LSU queue with shifted 16-B stores
    otherwise), the warp rings forced on (shifted stores out of shared memory for every byte
    offset) and the static slices; canary bytes outside the segments must survive."""
    p = 8
    rng = np.random.default_rng(7)
    counts = rng.integers(512 << 10, 3 << 19, size=(p, p)).astype(np.int64)
    counts[0, 3] = 0
    sc, rc = counts, counts.T.copy()
    gs = rng.integers(0, 16, size=(p, p))
    gr = rng.integers(0, 16, size=(p, p))
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc + gs, 1)[:, :-1]; sd += gs[:, :1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc + gr, 1)[:, :-1]; rd += gr[:, :1]
    S = int((sd + sc).max()) + 16
    R = int((rd + rc).max()) + 16
    send = rng.integers(0, 256, size=(p, S), dtype=np.uint8)
    recv0 = np.full((p, R), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 1, recv0)
    if not dyn:
        monkeypatch.setenv("MPXA_NO_DYN", "1")
    if dyn == "wring":      # every byte offset class through the warp rings' shifted stores
        monkeypatch.setenv("MPXA_WRING", "2")
    for G in (0, 8):
        c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, timeout_s=20.0)
        for off in (0, 1, 8):           # shift the whole send buffer: more alignment classes
            d_send = torch.zeros(p * S + 16, dtype=torch.uint8, device=DEV)
            d_send[off:off + p * S] = dev(send.reshape(-1))
            for algo in ("pairwise", "bruck"):
                d_recv = dev(recv0)
                c.alltoallv(d_send[off:off + p * S].view(p, S), sc, sd, d_recv, rc, rd, algo=algo)
                assert np.array_equal(host(d_recv), want), (G, off, dyn, algo)
        c.finalize()


def test_alltoallv_counts_kernel():
    """A2: single GPU -> fused transpose+scan kernel; emulated GPUs -> the multi-process
    path (alltoall of one int64 per pair through the flag protocol, then the scan kernel)."""
    for p in (1, 3, 8, 32, 40):
        sc = synth.cfg4_counts(p, p, 4096)
        rc_w, rd_w, _ = oracle.counts_exchange(sc)
        for G in [0] + [G for G in (2, 4, 8) if p % G == 0]:
            c = comm(p, G)
            d_sc = dev(sc)
            d_rc = torch.zeros_like(d_sc)
            d_rd = torch.zeros_like(d_sc)
            c.alltoallv_counts(d_sc, d_rc, d_rd)
            assert np.array_equal(host(d_rc), rc_w) and np.array_equal(host(d_rd), rd_w), (p, G)


# ------------------------------------------------------------------ persistent requests

def test_persistent_alltoallv_100_cycles():
    """cfg4: init once, start/wait 100 times; fresh data verified at cycles 0, 1, 99."""
    p = 8
    c4 = synth.cfg4_counts(0, p, 4096)
    for G in (0, 8):
        c = comm(p, G, 2)
        for algo in ("pairwise", "hier", "bruck"):
            send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(0, c4, elem=8)
            d_send = dev(send.view(np.int64))
            d_recv = torch.zeros((p, Rcap // 8), dtype=torch.int64, device=DEV)
            req = c.alltoallv_init(d_send, sc, sd, d_recv, rc, rd, algo=algo)
            assert req.algorithm == algo
            launches0 = c.launch_count()
            for cyc in range(100):
                if cyc in (0, 1, 99):
                    send_c, *_ = synth.alltoallv_buffers(cyc + 100, c4, elem=8)
                    d_send.copy_(dev(send_c.view(np.int64)))
                req.start()
                req.wait()
                if cyc in (0, 1, 99):
                    want = oracle.alltoallv_definition(send_c, sc, sd, rc, rd, 8, np.zeros((p, Rcap), np.uint8))
                    assert np.array_equal(host(d_recv).view(np.uint8), want), (G, algo, cyc)
            assert c.launch_count() - launches0 == 100      # one kernel per start, nothing else
            req.free()


def test_persistent_lifecycle_errors():
    p = 4
    c = comm(p)
    d_send = torch.zeros(p * p * 16, dtype=torch.uint8, device=DEV)
    d_recv = torch.zeros_like(d_send)
    req = c.alltoall_init(d_send, d_recv, algo="pairwise")
    with pytest.raises(MpxaError) as e:
        req.wait()                        # wait on INACTIVE
    assert e.value.status == M.ERR_LIFECYCLE
    req.start()
    with pytest.raises(MpxaError) as e:
        req.start()                       # start on ACTIVE
    assert e.value.status == M.ERR_LIFECYCLE
    with pytest.raises(MpxaError) as e:
        req.free()                        # free while ACTIVE
    assert e.value.status == M.ERR_LIFECYCLE
    req.wait()
    req.free()


@pytest.mark.parametrize("op", ["alltoall", "allgather"])
def test_persistent_uniform_cycles(op):
    p, b = 8, 4096 + 64
    for G in (0, 4):
        c = comm(p, G)
        for algo in M.list_algorithms(op):
            if op == "alltoall":
                send = synth.alltoall_sendbuf(1, p, b)
                d_send, d_recv = dev(send), torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
                req = c.alltoall_init(d_send, d_recv, algo=algo)
            else:
                send = synth.allgather_sendbuf(1, p, b)
                d_send, d_recv = dev(send), torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
                req = c.allgather_init(d_send, d_recv, algo=algo)
            for cyc in range(5):
                fresh = (synth.alltoall_sendbuf(cyc, p, b) if op == "alltoall"
                         else synth.allgather_sendbuf(cyc, p, b))
                d_send.copy_(dev(fresh))
                req.start()
                req.wait()
                want = (oracle.alltoall_definition(fresh) if op == "alltoall"
                        else oracle.allgather_definition(fresh))
                assert np.array_equal(host(d_recv), want), (G, algo, cyc)
            req.free()


def test_selector_and_registry():
    c = comm(8)
    assert c.get_algorithm("alltoall", 1 << 20) in ("pairwise", "bruck", "hier")
    c.set_algorithm("allgather", "ring")
    assert c.get_algorithm("allgather", 4) == "ring"
    c.set_algorithm("allgather", "default")
    c.set_algorithm("alltoallv", "bruck")             # Bruck-v (f2 iii) is selectable
    assert c.get_algorithm("alltoallv", 64) == "bruck"
    c.set_algorithm("alltoallv", "default")
    with pytest.raises(MpxaError):
        c.set_algorithm("alltoallv", "ring")          # ring is allgather-only
    # several ranks per GPU across GPUs: allgather beyond the eager range defaults to the
    # hierarchical variant (one NVLink copy per GPU instead of one per rank)
    ce = comm(32, 8, 4)
    assert ce.get_algorithm("allgather", 64) == "pairwise"
    assert ce.get_algorithm("allgather", 1 << 20) == "hier"
    assert ce.get_algorithm("alltoall", 1 << 20) == "pairwise"


# ------------------------------------------------------------------ full-size (bench launch config)

def _column_sample_check(send_d, recv_d, p, b, cols):
    """alltoall acts independently on every byte column of a block: check sampled columns
    through the oracle on the reduced (p, p*len(cols)) instance."""
    s = send_d.view(p, p, b)[:, :, cols].cpu().numpy().reshape(p, p * len(cols))
    r = recv_d.view(p, p, b)[:, :, cols].cpu().numpy().reshape(p, p * len(cols))
    assert np.array_equal(r, oracle.alltoall_definition(s))


@pytest.mark.parametrize("G", [0, 8])
def test_full_size_cfg3_p8_16MiB_sampled(G):
    p, b = 8, 16 << 20
    g = torch.Generator(device=DEV)
    g.manual_seed(0)
    send = torch.randint(0, 256, (p, p * b), dtype=torch.uint8, device=DEV, generator=g)
    recv = torch.zeros_like(send)
    rng = np.random.default_rng(0)
    cols = np.unique(np.concatenate([rng.integers(0, b, 4096), [0, 1, 15, 16, 127, 128, b - 1]]))
    c = comm(p, G, 2)
    for algo in ("pairwise", "bruck", "hier"):
        recv.zero_()
        c.alltoall(send, recv, algo=algo)
        torch.cuda.synchronize()
        _column_sample_check(send, recv, p, b, torch.from_numpy(cols).to(DEV))
        # whole-buffer invariant: recv is a permutation of blocks of send
        assert torch.equal(recv.view(p, p, b).transpose(0, 1).reshape(p, p * b), send)


def test_full_size_cfg2_allgather_64MiB_sampled():
    p, b = 8, 64 << 20
    g = torch.Generator(device=DEV)
    g.manual_seed(1)
    send = torch.randint(0, 256, (p, b), dtype=torch.uint8, device=DEV, generator=g)
    recv = torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
    c = comm(p)
    for algo in ("pairwise", "bruck", "ring"):
        recv.zero_()
        c.allgather(send, recv, algo=algo)
        torch.cuda.synchronize()
        cols = torch.from_numpy(np.unique(np.random.default_rng(2).integers(0, b, 4096))).to(DEV)
        s = send[:, cols].cpu().numpy()
        r = recv.view(p, p, b)[:, :, cols].cpu().numpy().reshape(p, -1)
        assert np.array_equal(r, oracle.allgather_definition(s)), algo
        for r_ in range(p):
            assert torch.equal(recv[r_].view(p, b), send), algo


def test_graph_replay_device_epochs():
    """CUDA-graph capture of several collectives, replayed repeatedly: epochs live on the
    device, so the emulated multi-GPU flag protocol stays consistent across replays."""
    p, b = 8, 4096 + 16
    for G in (0, 4, 8):
        c = comm(p, G, 2)
        for algo in ("pairwise", "bruck", "hier"):
            send = synth.alltoall_sendbuf(G, p, b)
            d_send = dev(send)
            d_recv = torch.zeros_like(d_send)
            s = torch.cuda.Stream()
            c.alltoall(d_send, d_recv, algo=algo, stream=s)      # compile + warm outside capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(3):
                    c.alltoall(d_send, d_recv, algo=algo, stream=s)
            for rep in range(4):
                fresh = synth.alltoall_sendbuf(100 + rep, p, b)
                d_send.copy_(dev(fresh))
                d_recv.zero_()
                torch.cuda.synchronize()
                g.replay()
                torch.cuda.synchronize()
                assert np.array_equal(host(d_recv), oracle.alltoall_definition(fresh)), (G, algo, rep)
            assert c.check() == 0
            del g


@pytest.mark.parametrize("p,b,G", [(32, 262144, 0), (16, 1 << 20, 0), (32, 1 << 20, 4), (16, (1 << 20) + 40, 0),
                                   (32, 65536, 0)])
def test_dynamic_mode_many_move_tiles(p, b, G):
    """Single-step launches with more moves than one shared-memory tile (p^2 > 128) run the
    dynamic executor tile by tile (one pair of queues per tile): whole buffers vs the oracle,
    alltoall and allgather, aligned and 8-byte-misaligned blocks."""
    c = comm(p, G)
    rng = np.random.default_rng(p + b)
    send = rng.integers(0, 256, size=(p, p * b), dtype=np.uint8)
    d_send = dev(send)
    d_recv = torch.full_like(d_send, 0xA5)
    want = oracle.alltoall_definition(send)
    c.alltoall(d_send, d_recv, algo="pairwise")
    assert np.array_equal(host(d_recv), want), (p, b, G)
    if b >= (1 << 20):    # multi-step dynamic mode (step barrier, per-GPU flags when G > 0)
        for algo in ("bruck", "hier"):
            d_recv.fill_(0xA5)
            c.alltoall(d_send, d_recv, algo=algo)
            assert np.array_equal(host(d_recv), want), (p, b, G, algo)
    ag = send[:, :b].copy()
    d_ag = torch.full((p, p * b), 0x5A, dtype=torch.uint8, device=DEV)
    c.allgather(dev(ag), d_ag, algo="pairwise")
    assert np.array_equal(host(d_ag), oracle.allgather_definition(ag)), (p, b, G)


def test_one_shot_alltoallv_program_cache():
    """One-shot alltoallv reuses the compiled program when the count/displacement matrices
    repeat, and evicts (least recently used) past 32 layouts: every call stays exact."""
    p = 8
    c = comm(p)
    layouts = [synth.cfg4_counts(seed, p, 512) for seed in range(40)]
    for rep in range(2):
        for seed, c4 in enumerate(layouts):
            send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(seed + 100 * rep, c4, elem=8, packed=bool(seed % 2))
            recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
            d_recv = dev(recv0)
            c.alltoallv(dev(send.view(np.int64)), sc, sd, d_recv.view(torch.int64), rc, rd)
            want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0)
            assert np.array_equal(host(d_recv), want), (rep, seed)


def test_alltoallv_device_counts_pipeline():
    """cfg4's "counts/displs exchanged then data" entirely on the device: sendcounts on the
    GPU -> mpxa_alltoallv_counts (A2) -> recvcounts / rdispls on the GPU -> alltoallv and the
    persistent init taking the device arrays (copied by the library)."""
    p = 8
    c4 = synth.cfg4_counts(3, p, 4096)
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(3, c4, elem=8, packed=True)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, np.zeros((p, Rcap), np.uint8))
    for G in (0, 2):
        c = comm(p, G)
        d_sc = dev(sc)
        d_rc, d_rd = torch.zeros_like(d_sc), torch.zeros_like(d_sc)
        c.alltoallv_counts(d_sc, d_rc, d_rd)
        d_sd = dev(sd)
        d_recv = torch.zeros((p, Rcap // 8), dtype=torch.int64, device=DEV)
        c.alltoallv(dev(send.view(np.int64)), d_sc, d_sd, d_recv, d_rc, d_rd)
        assert np.array_equal(host(d_recv).view(np.uint8), want), G
        d_recv.zero_()
        req = c.alltoallv_init(dev(send.view(np.int64)), d_sc, d_sd, d_recv, d_rc, d_rd)
        req.start(); req.wait()
        assert np.array_equal(host(d_recv).view(np.uint8), want), G
        req.free()


@pytest.mark.parametrize("G", [0, 2])
def test_small_sync_mode_multistep(G):
    """Multi-step programs with short moves but more pieces than one CTA holds run the
    small-message kernel on several CTAs with a barrier per step (allgather Bruck / ring,
    hierarchical and Bruck alltoallv at mid sizes): exact vs the oracle."""
    p = 8
    c = comm(p, G, 2)
    for b in (1024, 4096 + 8, 65536):
        ag = np.random.default_rng(b).integers(0, 256, size=(p, b), dtype=np.uint8)
        want = oracle.allgather_definition(ag)
        for algo in ("bruck", "ring"):
            d_r = torch.full((p, p * b), 0x5A, dtype=torch.uint8, device=DEV)
            c.allgather(dev(ag), d_r, algo=algo)
            assert np.array_equal(host(d_r), want), (b, algo, G)
    c4 = synth.cfg4_counts(5, p, 16384)
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(5, c4, elem=8, packed=False)
    recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0)
    for algo in ("hier", "bruck"):
        d_recv = dev(recv0)
        c.alltoallv(dev(send.view(np.int64)), sc, sd, d_recv.view(torch.int64), rc, rd, algo=algo)
        assert np.array_equal(host(d_recv), want), (algo, G)


@pytest.mark.parametrize("G", [0, 2, 4])
def test_small_owned_flow_mode_multistep(G):
    """Uniform multi-step programs (Bruck, hierarchical, ring) with short moves on several
    CTAs, each owning the same flows in every step (no barrier): exact vs the oracle, on one
    device and across emulated GPUs (per-CTA flags)."""
    p = 8
    c = comm(p, G, 2)
    for b in (1024, 4096 + 4, 16384):
        send = np.random.default_rng(b).integers(0, 256, size=(p, p * b), dtype=np.uint8)
        want = oracle.alltoall_definition(send)
        for algo in ("bruck", "hier", "pairwise"):
            d_r = torch.full((p, p * b), 0xA5, dtype=torch.uint8, device=DEV)
            c.alltoall(dev(send), d_r, algo=algo)
            assert np.array_equal(host(d_r), want), (b, algo, G)


@pytest.mark.parametrize("p,G", [(8, 0), (8, 2), (8, 8), (32, 0), (32, 4)])
def test_small_variable_piece_mode(p, G):
    """Moves of very different lengths (mostly 1-3 byte segments, a few of ~60 KiB, byte
    misaligned): the small kernel counts 16-B pieces exactly per tile of moves (block scan)
    instead of max-move slots per move -- one-step (pairwise) and multi-step (Bruck, hier)
    programs, several tiles at p=32; exact vs the oracle, canaries intact."""
    rng = np.random.default_rng(p * 10 + G)
    counts = rng.integers(0, 4, size=(p, p)).astype(np.int64)
    big = rng.choice(p * p, size=4, replace=False)
    counts.reshape(-1)[big] = rng.integers(50 << 10, 60 << 10, size=4)
    sc, rc = counts, counts.T.copy()
    gs = rng.integers(0, 16, size=(p, p))
    gr = rng.integers(0, 16, size=(p, p))
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc + gs, 1)[:, :-1]; sd += gs[:, :1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc + gr, 1)[:, :-1]; rd += gr[:, :1]
    S = int((sd + sc).max()) + 16
    R = int((rd + rc).max()) + 16
    send = rng.integers(0, 256, size=(p, S), dtype=np.uint8)
    recv0 = np.full((p, R), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 1, recv0)
    c = comm(p, G, 2)
    for algo in ("pairwise", "bruck", "hier"):
        d_recv = dev(recv0)
        c.alltoallv(dev(send), sc, sd, d_recv, rc, rd, algo=algo)
        assert np.array_equal(host(d_recv), want), (algo, G)
    # persistent request first started inside a CUDA-graph capture: the split companion
    # program cannot be uploaded there, the variable-piece kernel runs on the original moves;
    # a later eager start builds the companion -- both exact
    d_send, d_recv = dev(send), dev(recv0)
    req = c.alltoallv_init(d_send, sc, sd, d_recv, rc, rd, algo="bruck")
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        req.start(s); req.wait(s)
    for rep in range(2):
        d_recv.copy_(dev(recv0)); torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        assert np.array_equal(host(d_recv), want), ("graph", rep, G)
        d_recv.copy_(dev(recv0)); torch.cuda.synchronize()
        req.start(); req.wait(); torch.cuda.synchronize()
        assert np.array_equal(host(d_recv), want), ("eager", rep, G)
    del g
    req.free()
    assert c.check() == 0


@pytest.mark.parametrize("G", [2, 4, 8])
def test_eager_ll_mode_interleaved(G):
    """Eager (LL) launches -- payload words carry the launch's flag in the receiver's staging,
    two parities alternating per eager launch -- interleaved with CTS-mode launches (large
    blocks) and with pairs that exchange nothing (flag-only words): every result exact, many
    launches in a row so both parities are reused."""
    p = 8
    c = comm(p, G, 2)
    rng = np.random.default_rng(G)
    for it in range(12):
        b = int(rng.choice([16, 100, 4096 + 4, 300_000]))     # 300 KB: CTS mode, not eager
        send = synth.alltoall_sendbuf(it * 7 + G, p, b)
        algo = ("pairwise", "bruck", "hier")[it % 3]
        got = run_alltoall(c, send, algo)
        assert np.array_equal(got, oracle.alltoall_definition(send)), (it, b, algo)
        ag = rng.integers(0, 256, size=(p, 24 + it), dtype=np.uint8)
        d_r = torch.full((p, p * ag.shape[1]), 0x5A, dtype=torch.uint8, device=DEV)
        c.allgather(dev(ag), d_r, algo=("pairwise", "bruck", "ring")[it % 3])
        assert np.array_equal(host(d_r), oracle.allgather_definition(ag)), it
    # sparse alltoallv: most GPU pairs exchange nothing (flag-only words), byte-granular
    counts = np.zeros((p, p), np.int64)
    counts[0, 5] = 37
    counts[3, 3] = 11
    counts[6, 1] = 4
    sc, rc = counts, counts.T.copy()
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
    S, R = int((sd + sc).max()) + 8, int((rd + rc).max()) + 8
    send = rng.integers(0, 256, size=(p, S), dtype=np.uint8)
    recv0 = np.full((p, R), 0xA5, dtype=np.uint8)
    want = oracle.alltoallv_definition(send, sc, sd, rc, rd, 1, recv0)
    for rep in range(3):
        d_recv = dev(recv0)
        c.alltoallv(dev(send), sc, sd, d_recv, rc, rd, algo="pairwise")
        assert np.array_equal(host(d_recv), want), rep
    assert c.check() == 0


@pytest.mark.parametrize("G", [2, 4, 8])
def test_direct_protocol_small_sizes(G, monkeypatch):
    """MPXA_NO_LL=1: small multi-GPU launches through the direct protocol (CTS + per-step
    flags, small kernel) -- the path eager mode replaced for these sizes stays exact."""
    p = 8
    monkeypatch.setenv("MPXA_NO_LL", "1")
    c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=2, timeout_s=20.0)
    for b in (1, 16, 260, 4096 + 12):
        send = synth.alltoall_sendbuf(b + G, p, b)
        want = oracle.alltoall_definition(send)
        for algo in ("pairwise", "bruck", "hier"):
            assert np.array_equal(run_alltoall(c, send, algo), want), (b, algo)
            assert "eager" not in c.last_launch_path()
        ag = np.random.default_rng(b).integers(0, 256, size=(p, b), dtype=np.uint8)
        for algo in ("pairwise", "bruck", "ring"):
            d_r = torch.full((p, p * b), 0x5A, dtype=torch.uint8, device=DEV)
            c.allgather(dev(ag), d_r, algo=algo)
            assert np.array_equal(host(d_r), oracle.allgather_definition(ag)), (b, algo)
    assert c.check() == 0
    c.finalize()


@pytest.mark.skipif(any(os.environ.get(k, "0") != "0" for k in ("MPXA_NO_LL", "MPXA_NO_DYN", "MPXA_NO_TINY")),
                    reason="asserts the default execution paths")
def test_execution_paths_are_the_intended_ones(monkeypatch):
    """The launches these parity tests rely on take the paths they are meant to exercise
    (mpxa__last_launch): eager on emulated GPUs for small messages, direct otherwise; the
    variable-piece mode for mixed move lengths; dynamic queues for a large allgather; the
    small kernel's owned-flow / sync modes for multi-step mid sizes; shared-memory WORK for a
    one-CTA single-GPU Bruck."""
    p = 8
    c1 = comm(p, 0, 2)
    send = synth.alltoall_sendbuf(1, p, 16)
    run_alltoall(c1, send, "bruck")          # one CTA, several steps, one GPU: the tiny kernel
    assert {"small", "tiny"} <= c1.last_launch_path() and "eager" not in c1.last_launch_path()
    monkeypatch.setenv("MPXA_NO_TINY", "1")   # the general kernel: WORK rows in shared memory
    cg = Comm(ranks_per_proc=p, device=0, group_size=2, timeout_s=20.0)
    assert np.array_equal(run_alltoall(cg, send, "bruck"), oracle.alltoall_definition(send))
    assert {"small", "swork"} <= cg.last_launch_path() and "tiny" not in cg.last_launch_path()
    cg.finalize()
    monkeypatch.delenv("MPXA_NO_TINY")
    # mid-size multi-step on one GPU: the tiny kernel over several CTAs owning flows
    ag4 = np.random.default_rng(4).integers(0, 256, size=(p, 4096 + 8), dtype=np.uint8)
    d_r4 = torch.full((p, p * ag4.shape[1]), 0x5A, dtype=torch.uint8, device=DEV)
    for algo in ("ring", "bruck"):
        c1.allgather(dev(ag4), d_r4, algo=algo)
        assert {"small", "tiny", "own"} <= c1.last_launch_path(), algo
        assert np.array_equal(host(d_r4), oracle.allgather_definition(ag4)), algo
    c4 = comm(p, 4, 2)
    run_alltoall(c4, send, "pairwise")
    assert {"small", "eager"} <= c4.last_launch_path()
    big = synth.alltoall_sendbuf(2, p, 300_000)
    run_alltoall(c4, big, "pairwise")
    assert "eager" not in c4.last_launch_path()
    # mixed lengths: variable pieces
    counts = np.ones((p, p), np.int64)
    counts[0, 1] = 60 << 10
    counts[2, 3] = 50 << 10
    sc, rc = counts, counts.T.copy()
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
    S, R = int((sd + sc).max()), int((rd + rc).max())
    sendv = np.random.default_rng(0).integers(0, 256, size=(p, S), dtype=np.uint8)
    d_r = torch.zeros((p, R), dtype=torch.uint8, device=DEV)
    c1.alltoallv(dev(sendv), sc, sd, d_r, rc, rd, algo="pairwise")
    assert {"small", "var"} <= c1.last_launch_path()
    assert np.array_equal(host(d_r), oracle.alltoallv_definition(sendv, sc, sd, rc, rd, 1, np.zeros((p, R), np.uint8)))
    # large allgather: dynamic work queues in the executor
    ag = torch.randint(0, 256, (p, 8 << 20), dtype=torch.uint8, device=DEV)
    out = torch.empty((p, p * (8 << 20)), dtype=torch.uint8, device=DEV)
    c1.allgather(ag, out, algo="pairwise")
    assert "dyn" in c1.last_launch_path() and c1.last_launch_path() <= {"dyn", "wring"}   # (wring: MPXA_WRING=2)
    del ag, out


def test_cooperative_launches_where_ctas_wait_on_each_other():
    """Launches whose CTAs wait on one another are cooperative (co-residency guaranteed, with
    PDL): several steps over several CTAs on one GPU (per-step row barriers) and emulated GPUs;
    one-step and owned-flow launches are not (mpxa__last_launch bit "coop")."""
    p = 8
    c1 = comm(p, 0, 2)
    small = synth.alltoall_sendbuf(1, p, 16)
    run_alltoall(c1, small, "pairwise")
    assert "coop" not in c1.last_launch_path()
    big = synth.alltoall_sendbuf(3, p, 1 << 20)            # Bruck, 1 MiB blocks: multi-step executor
    assert np.array_equal(run_alltoall(c1, big, "bruck"), oracle.alltoall_definition(big))
    path = c1.last_launch_path()
    assert "coop" in path and "tiny" not in path and "own" not in path, sorted(path)
    c4 = synth.cfg4_counts(5, p, 64 << 10, elem=8)          # hierarchical alltoallv: sync mode
    send, sc, sd, rc, rd, S, Rcap = synth.alltoallv_buffers(5, c4, elem=8, packed=True)
    recv0 = np.full((p, Rcap), 0xA5, dtype=np.uint8)
    d_r = dev(recv0)
    c1.alltoallv(dev(send), sc, sd, d_r, rc, rd, algo="hier", dtype_size=8)
    path = c1.last_launch_path()
    assert np.array_equal(host(d_r), oracle.alltoallv_definition(send, sc, sd, rc, rd, 8, recv0))
    assert ("sync" in path) <= ("coop" in path), sorted(path)
    ce = comm(p, 4, 2)
    run_alltoall(ce, small, "pairwise")
    assert "coop" in ce.last_launch_path()


@pytest.mark.skipif(os.environ.get("MPXA_NO_LL", "0") != "0", reason="asserts the eager path")
def test_eager_persistent_first_start_captured():
    """A persistent request's eager companion is built at *_init, so even a first start()
    inside a CUDA-graph capture runs eager (the same in every process); replays exact."""
    p, G, b = 8, 4, 1000
    c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=2, timeout_s=20.0)
    send = synth.alltoall_sendbuf(9, p, b)
    d_s, d_r = dev(send), torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
    req = c.alltoall_init(d_s, d_r, algo="pairwise")
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        req.start(s); req.wait(s)
    assert "eager" in c.last_launch_path()
    for rep in range(3):
        fresh = synth.alltoall_sendbuf(20 + rep, p, b)
        d_s.copy_(dev(fresh)); d_r.zero_(); torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        assert np.array_equal(host(d_r), oracle.alltoall_definition(fresh)), rep
    del g
    req.free()
    assert c.check() == 0
    c.finalize()


@pytest.mark.parametrize("G", [2, 4])
def test_two_sizes_one_program_graph_replay(G):
    """Two persistent requests of the same (op, variant) at different sizes share one cached
    program but need different eager companions.  Capture start(Y) in a graph, run X eagerly
    (plus one-shot calls at a third size), replay Y: the graph's companion must still be
    alive and the replay exact (a companion replaced per unit was freed under
    the graph)."""
    p = 8
    c = Comm(ranks_per_proc=p, device=0, emulate_gpus=G, group_size=2, timeout_s=20.0)
    bx, by, bz = 200, 1000, 48
    sx, sy = synth.alltoall_sendbuf(31, p, bx), synth.alltoall_sendbuf(32, p, by)
    dx_s, dx_r = dev(sx), torch.zeros((p, p * bx), dtype=torch.uint8, device=DEV)
    dy_s, dy_r = dev(sy), torch.zeros((p, p * by), dtype=torch.uint8, device=DEV)
    rx = c.alltoall_init(dx_s, dx_r, algo="pairwise")
    ry = c.alltoall_init(dy_s, dy_r, algo="pairwise")
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ry.start(s); ry.wait(s)
    for rep in range(3):
        rx.start(); rx.wait()
        sz = synth.alltoall_sendbuf(40 + rep, p, bz)
        assert np.array_equal(run_alltoall(c, sz, "pairwise"), oracle.alltoall_definition(sz)), rep
        assert np.array_equal(host(dx_r), oracle.alltoall_definition(sx)), rep
        fresh = synth.alltoall_sendbuf(50 + rep, p, by)
        dy_s.copy_(dev(fresh)); dy_r.zero_(); torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        assert np.array_equal(host(dy_r), oracle.alltoall_definition(fresh)), ("replay", rep)
    del g
    rx.free(); ry.free()
    assert c.check() == 0
    c.finalize()


@pytest.mark.parametrize("G", [0, 4])
def test_many_ranks_beyond_rank_table(G):
    """p = 300 ranks (beyond the small kernel's 256-entry rank-base table: bases computed per
    piece, no resolved moves / eager companion): pairwise, Bruck and hier alltoall and the
    allgathers stay exact, on one device and over 4 emulated GPUs."""
    p = 300
    c = comm(p, G, 4)
    for b in (4, 36):
        send = synth.alltoall_sendbuf(b, p, b)
        want = oracle.alltoall_definition(send)
        for algo in ("pairwise", "bruck", "hier"):
            assert np.array_equal(run_alltoall(c, send, algo), want), (b, algo)
        ag = np.random.default_rng(b).integers(0, 256, size=(p, b), dtype=np.uint8)
        for algo in ("pairwise", "bruck", "ring"):
            d_r = torch.full((p, p * b), 0x5A, dtype=torch.uint8, device=DEV)
            c.allgather(dev(ag), d_r, algo=algo)
            assert np.array_equal(host(d_r), oracle.allgather_definition(ag)), (b, algo)
    assert c.check() == 0


def test_persistent_wait_on_another_stream():
    """mpxa_wait on a stream other than the start stream orders that stream after the
    collective (the start stream is delayed by a long device sleep before the start): a copy
    of recvbuf queued on the wait stream right after the wait sees the whole result."""
    p, b = 8, 4096
    c = comm(p)
    send = synth.alltoall_sendbuf(77, p, b)
    d_s, d_r = dev(send), torch.zeros((p, p * b), dtype=torch.uint8, device=DEV)
    req = c.alltoall_init(d_s, d_r, algo="pairwise")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = torch.zeros_like(d_r)
    for rep in range(3):
        d_r.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            torch.cuda._sleep(50_000_000)             # the collective starts late on s1
        req.start(s1)
        req.wait(s2)
        with torch.cuda.stream(s2):
            out.copy_(d_r)
        torch.cuda.synchronize()
        assert np.array_equal(host(out), oracle.alltoall_definition(send)), rep
    req.free()
    assert c.check() == 0

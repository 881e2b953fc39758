"""CPU simulator of libmpxa schedules (test utility).

Executes the moves of a compiled plan (include/mpxa_plan.h) on numpy buffers, step by
step, with the executor's semantics, and checks the properties the sm_100a kernel relies
on:
  * within a step no byte is written twice and no byte written in the step is also read
    in it (moves of one step run concurrently on the GPU);
  * every read of a library-workspace or recv region written earlier in the same launch
    covers exactly the interval a single earlier move wrote, with the same flow (CTA
    ownership: the CTA that reads slice c of a flow is the CTA that wrote it);
  * every workspace / recv byte is written at most once per launch (so no CTA can overwrite
    data that a CTA owning another flow has still to read: no cross-CTA WAR hazard);
  * a GPU only executes moves whose source rank it owns (push model), and a step's
    signal/wait masks cover every cross-GPU write.
"""
import numpy as np

SEND, RECV, WORK = 0, 1, 2


def simulate(plan, send, recv, unit, work_units=None):
    """send/recv: (p, bytes) uint8 arrays (rank rows); returns recv (modified copy)."""
    p, R, G = plan.p, plan.R, plan.G
    wu = plan.info["work_units"] if work_units is None else work_units
    work = np.zeros((p, max(1, wu * unit)), dtype=np.uint8)
    recv = recv.copy()
    bufs = {SEND: send, RECV: recv, WORK: work}
    steps = [plan.steps(g) for g in range(G)]
    moves = [plan.moves(g) for g in range(G)]
    nsteps = len(steps[0])
    assert all(len(s) == nsteps for s in steps)
    written = {}          # (kind, rank) -> {offset: length} intervals written this launch
    flows = {}            # (kind, rank, offset) -> flow of the data written there
    ever_written = set()  # (kind, rank, byte) written in this launch
    for s in range(nsteps):
        reads, writes = [], []
        sig = [0] * G
        wt = [0] * G
        for g in range(G):
            st = steps[g][s]
            fl = [m.flow for m in moves[g][st.move_begin:st.move_end]]
            assert fl == sorted(fl), "moves of a step must be sorted by flow"
            assert max(fl, default=0) < plan.info["nflows"]
            for m in moves[g][st.move_begin:st.move_end]:
                assert m.src_rank // R == g, "move executed by a GPU that does not own its source"
                if m.src_kind != SEND:
                    assert flows.get((m.src_kind, m.src_rank, m.src_off * unit)) == m.flow, "flow not preserved"
                dst_ranks = range(p) if m.fanout else [m.dst_rank]
                src = (m.src_kind, m.src_rank, m.src_off * unit, m.len * unit)
                reads.append(src)
                for d in dst_ranks:
                    writes.append(((m.dst_kind, d, m.dst_off * unit, m.len * unit), src))
                    if d // R != g:
                        sig[g] |= 1 << (d // R)
                        wt[d // R] |= 1 << g
        for g in range(G):
            assert steps[g][s].signal_mask == sig[g] and steps[g][s].wait_mask == wt[g], "signal/wait masks"
        # hazards inside the step
        wmap = {}
        for (k, r, o, n), _ in writes:
            for b in range(o, o + n):
                key = (k, r, b)
                assert key not in wmap, f"byte written twice in step {s}: {key}"
                wmap[key] = True
        for (k, r, o, n) in reads:
            if k == SEND:
                continue
            assert not any((k, r, b) in wmap for b in range(o, o + n)), f"read-after-write in step {s}"
            prev = written.get((k, r), {})
            if n:
                assert prev.get(o) == n, f"read of ({k},{r},{o},{n}) not matching one earlier write"
        # apply: snapshot sources, then write
        data = [(dst, bufs[sk][sr, so:so + sn].copy()) for (dst, (sk, sr, so, sn)) in writes]
        for g in range(G):
            st = steps[g][s]
            for m in moves[g][st.move_begin:st.move_end]:
                if not m.fanout:
                    flows[(m.dst_kind, m.dst_rank, m.dst_off * unit)] = m.flow
        for (dk, dr, do, dn), val in data:
            for b in range(do, do + dn):
                assert (dk, dr, b) not in ever_written, f"byte written twice in one launch: {(dk, dr, b)}"
                ever_written.add((dk, dr, b))
            bufs[dk][dr, do:do + dn] = val
            written.setdefault((dk, dr), {})[do] = dn
    return recv


LL = 3            # eager staging (mpxa_plan_eager)
LL_WORDS = 32768  # kLLWords (mpxa_internal.h): staging words per (parity, source GPU)


def simulate_eager(plan, send, recv, unit, work_units=None):
    """Execute an eager (LL) plan (Plan.eager) with the kernel's semantics: per step, every
    GPU first runs its local moves and SEND moves (payload -> 4-byte words of the (src, dst)
    stream), then its RECEIVE moves (words -> destination).  Checks: receives are the last
    moves of each step and their number is the step's wait_mask; a GPU reads only its own
    sources and writes only its own ranks; every staging word is written once per launch and
    read only after it was written (same or earlier step); streams fit LL_WORDS; every
    ordered GPU pair exchanges at least one word (the parity invariant).  Returns recv."""
    p, R, G = plan.p, plan.R, plan.G
    wu = plan.info["work_units"] if work_units is None else work_units
    work = np.zeros((p, max(1, wu * unit)), dtype=np.uint8)
    recv = recv.copy()
    bufs = {SEND: send, RECV: recv, WORK: work}
    staging = {}      # (src gpu, dst gpu) -> bytearray of payload (4 bytes per word)
    wrote = {}        # (src gpu, dst gpu) -> set of word indexes written
    steps = [plan.steps(g) for g in range(G)]
    moves = [plan.moves(g) for g in range(G)]
    nsteps = len(steps[0])

    def words(m):
        return max(1, (m.len * unit + 3) // 4)

    def own_ranks(g):
        return range(g * R, (g + 1) * R)

    for s in range(nsteps):
        phase_b = []
        for g in range(G):
            st = steps[g][s]
            mv = moves[g][st.move_begin:st.move_end]
            nrecv = st.wait_mask
            assert st.signal_mask == 0
            assert all(m.src_kind == LL for m in mv[len(mv) - nrecv:]), "receives last"
            assert not any(m.src_kind == LL for m in mv[:len(mv) - nrecv])
            for m in mv[:len(mv) - nrecv]:
                assert m.src_rank // R == g, "a GPU reads only its own ranks"
                data = bufs[m.src_kind][m.src_rank, m.src_off * unit:(m.src_off + m.len) * unit].copy()
                if m.dst_kind == LL:
                    d = m.dst_rank
                    assert d != g and m.fanout == 0
                    buf = staging.setdefault((g, d), bytearray(4 * LL_WORDS))
                    ws = wrote.setdefault((g, d), set())
                    for w in range(m.dst_off, m.dst_off + words(m)):
                        assert w < LL_WORDS and w not in ws, "staging word written twice"
                        ws.add(w)
                    buf[4 * m.dst_off:4 * m.dst_off + len(data)] = data.tobytes()
                else:
                    targets = own_ranks(g) if m.fanout == 2 else [m.dst_rank]
                    assert m.fanout in (0, 2)
                    for r in targets:
                        assert r // R == g, "a local move writes only this GPU's ranks"
                        bufs[m.dst_kind][r, m.dst_off * unit:(m.dst_off + m.len) * unit] = data
            phase_b.append((g, mv[len(mv) - nrecv:]))
        for g, mv in phase_b:
            for m in mv:
                src = m.src_rank
                ws = wrote.get((src, g), set())
                for w in range(m.src_off, m.src_off + words(m)):
                    assert w in ws, "word received before it was sent"
                n = m.len * unit
                data = np.frombuffer(bytes(staging[(src, g)][4 * m.src_off:4 * m.src_off + n]), np.uint8)
                targets = own_ranks(g) if m.fanout == 2 else [m.dst_rank]
                for r in targets:
                    assert r // R == g
                    bufs[m.dst_kind][r, m.dst_off * unit:m.dst_off * unit + n] = data
    for a in range(G):
        for b in range(G):
            if a != b:
                assert wrote.get((a, b)), f"GPU pair {a}->{b} exchanges no word"
    return recv

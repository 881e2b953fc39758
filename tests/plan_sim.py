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

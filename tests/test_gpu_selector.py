"""A10 variant selection ("select a default algorithm, but make all
implementations publicly available"), -m gpu.

The default variant of a call is: mpxa_set_algorithm override > the measured selector table >
built-in fallback rules.  These tests load tables and check the per-size choice through
mpxa_get_algorithm and through what a default-variant persistent request actually runs;
they also check the shipped table (paper_2309_07337_b200/selector_b200.txt, written by
bench.py --write-selector from B200 measurements) parses and is what a fresh comm uses.
Which variant is fastest is performance only ("parity unpinned"): every
choice is bit-identical, which the parity suites check."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2309_07337_b200 import Comm, MpxaError  # noqa: E402
from paper_2309_07337_b200 import mpxa as M  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIPPED = os.path.join(ROOT, "paper_2309_07337_b200", "selector_b200.txt")
BIG = 18446744073709551615


def _table(tmp_path, lines):
    f = tmp_path / "sel.txt"
    f.write_text("# test table\n" + "\n".join(lines) + "\n")
    return str(f)


def test_table_choices_per_size(tmp_path):
    c = Comm(ranks_per_proc=8, device=0)           # p = 8, R = 8, G = 1, g = 8
    c.load_selector(_table(tmp_path, [
        "alltoall 8 8 1 8 1024 bruck",
        "alltoall 8 8 1 8 65536 hier",
        f"alltoall 8 8 1 8 {BIG} pairwise",
        "allgather 8 8 1 8 4096 ring",
        f"allgather 8 8 1 8 {BIG} bruck",
        "alltoallv 8 8 1 8 100 bruck",
        "allgather 8 8 2 4 1024000 pairwise",       # another G / g: never matches this comm
    ]))
    for b, want in ((1, "bruck"), (1024, "bruck"), (1025, "hier"), (65536, "hier"), (65537, "pairwise"),
                    (1 << 30, "pairwise")):
        assert c.get_algorithm("alltoall", b) == want, b
    for b, want in ((4, "ring"), (4096, "ring"), (4097, "bruck")):
        assert c.get_algorithm("allgather", b) == want, b
    assert c.get_algorithm("alltoallv", 64) == "bruck"
    assert c.get_algorithm("alltoallv", 101) == "pairwise"      # no row: fallback rule
    # what a default-variant request runs
    for b, want in ((512, "bruck"), (4096, "hier"), (1 << 20, "pairwise")):
        s = torch.zeros((8, 8 * b), dtype=torch.uint8, device="cuda")
        r = torch.zeros_like(s)
        q = c.alltoall_init(s, r)
        assert q.algorithm == want, b
        q.free()
    # the override beats the table
    c.set_algorithm("alltoall", "pairwise")
    assert c.get_algorithm("alltoall", 1) == "pairwise"
    c.set_algorithm("alltoall", None)
    assert c.get_algorithm("alltoall", 1) == "bruck"
    c.finalize()


def test_alltoallv_selection_uses_global_mean(tmp_path):
    """A v-collective's table size is the mean pair segment of the global count matrix."""
    c = Comm(ranks_per_proc=4, device=0)
    c.load_selector(_table(tmp_path, ["alltoallv 4 4 1 4 64 bruck", f"alltoallv 4 4 1 4 {BIG} hier"]))
    for mean, want in ((8, "bruck"), (512, "hier")):        # int64 elements: 64 B vs 4 KiB mean
        counts = np.full((4, 4), mean, np.int64)
        sd = np.arange(4, dtype=np.int64)[None, :].repeat(4, 0) * mean
        s = torch.zeros((4, 4 * mean * 8), dtype=torch.uint8, device="cuda")
        r = torch.zeros_like(s)
        q = c.alltoallv_init(s, counts, sd, r, counts, sd, dtype_size=8)
        assert q.algorithm == want, mean
        q.free()
    c.finalize()


def test_five_field_rows_match_any_topology(tmp_path):
    path = _table(tmp_path, ["alltoall 8 8 2048 bruck", f"alltoall 8 8 {BIG} pairwise"])
    for G, g in ((0, 0), (2, 2), (4, 4)):
        c = Comm(ranks_per_proc=8, device=0, emulate_gpus=G, group_size=g)
        c.load_selector(path)
        assert c.get_algorithm("alltoall", 2048) == "bruck" and c.get_algorithm("alltoall", 2049) == "pairwise"
        c.finalize()


def test_bad_tables_rejected(tmp_path):
    c = Comm(ranks_per_proc=4, device=0)
    for bad in ("alltoall 4 4 1 4 64 ring",          # alltoall has no ring
                "broadcast 4 4 64 pairwise",          # unknown op
                "alltoall 4 4 1 64 pairwise"):        # 6 fields
        with pytest.raises(MpxaError) as e:
            c.load_selector(_table(tmp_path, [bad]))
        assert e.value.status == M.ERR_ARG, bad
    c.finalize()


def test_shipped_table_is_loaded_and_used():
    """The measured table next to libmpxa.so: every row parses, and a fresh comm of each
    single-GPU configuration it covers returns the row's choice at the row's size."""
    rows = []
    for ln in open(SHIPPED):
        s = ln.split("#")[0].split()
        if s:
            assert len(s) == 7, ln
            rows.append((s[0], int(s[1]), int(s[2]), int(s[3]), int(s[4]), int(s[5]), s[6]))
    assert rows, "empty selector table"
    seen = set()
    for op, p, R, G, g, mb, algo in rows:
        if p != R or (G > 1 and p % G):     # single-process configurations (all ranks here)
            continue
        c = Comm(ranks_per_proc=R, device=0, emulate_gpus=G if G > 1 else 0, group_size=g)
        assert c.get_algorithm(op, min(mb, 1 << 40)) == algo, (op, p, R, G, g, mb)
        seen.add((op, p, G))
        c.finalize()
    assert ("alltoall", 8, 1) in seen and ("allgather", 8, 1) in seen

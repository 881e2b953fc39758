"""Host logic of bench.py (-m "not gpu"): the measured selector rows (per size the fastest
variant; a non-default one only when > 3 % faster than pairwise), the merge
into an existing table (numeric order inside a key, other keys kept), and the host-baseline
record (threaded oracle run, core counts, CPU model)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_selector_rows_choose_fastest_with_margin():
    var = {"pairwise": [(4, 10.0), (64, 10.0), (1024, 10.0), (4096, 10.0)],
           "bruck": [(4, 5.0), (64, 9.8), (1024, 12.0), (4096, 7.0)]}
    rows = bench.selector_rows("alltoall", 8, 8, 1, 8, var)
    # 4 B: bruck (2x faster); 64 B: within 3 % -> pairwise; 1 KiB: pairwise; 4 KiB: bruck
    assert rows == ["alltoall 8 8 1 8 4 bruck", "alltoall 8 8 1 8 1024 pairwise",
                    "alltoall 8 8 1 8 18446744073709551615 bruck"]


def test_write_selector_merges_and_orders_numerically(tmp_path):
    path = tmp_path / "sel.txt"
    path.write_text("# old\nallgather 8 8 1 8 18446744073709551615 ring\n"
                    "alltoall 8 8 1 8 18446744073709551615 bruck\n")
    bench.write_selector(["alltoall 8 8 1 8 18446744073709551615 pairwise", "alltoall 8 8 1 8 256 hier",
                          "alltoall 8 8 1 8 64 bruck"], str(path))
    rows = [ln for ln in path.read_text().splitlines() if ln and not ln.startswith("#")]
    assert rows == ["allgather 8 8 1 8 18446744073709551615 ring",       # other key kept
                    "alltoall 8 8 1 8 64 bruck", "alltoall 8 8 1 8 256 hier",
                    "alltoall 8 8 1 8 18446744073709551615 pairwise"]    # replaced, numeric order


def test_measured_selector_from_bench_records():
    sw = {"allgather": {"pairwise": [[4, 2.0, 1.0, 0.1], [8, 2.0, 1.0, 0.1]],
                        "bruck": [[4, 1.0, 1.0, 0.1], [8, 3.0, 1.0, 0.1]],
                        "torch_copy_baseline": [[4, 0.5, 1.0], [8, 0.5, 1.0]]},
          "alltoall": {"pairwise": [[4, 2.0, 1.0, 0.1]], "hier": [[4, 2.1, 1.0, 0.1]]}}
    cfgs = {"cfg4_alltoallv_p8_persistent_100x": {
        "mean_64B": {"variants_graph_us": {"pairwise": 2.0, "bruck": 5.0, "hier": 2.3}},
        "mean_4194304B": {"variants_graph_us": {"pairwise": 90.0, "bruck": 240.0, "hier": 80.0}}}}
    rows = bench.measured_selector(sw, cfgs, 8, 8, 8)
    assert "allgather 8 8 1 8 4 bruck" in rows and "allgather 8 8 1 8 18446744073709551615 pairwise" in rows
    assert "alltoall 8 8 1 8 18446744073709551615 pairwise" in rows          # torch baseline ignored
    assert rows[-2:] == ["alltoallv 8 8 1 8 64 pairwise", "alltoallv 8 8 1 8 18446744073709551615 hier"]


def test_cpu_baseline_record():
    send = np.random.default_rng(0).integers(0, 256, size=(4, 4096), dtype=np.uint8)
    d = bench.cpu_oracle_sample(send, 0.2)
    assert d["kind"] == "oracle" and d["unit"] == "GB/s" and d["value"] > 0
    assert 1 <= d["cores"] <= 4 and d["single_thread"]["cores"] == 1
    assert d["os_cpu_count"] >= 1 and d["affinity_cores"] >= 1


def test_schedule_units_closed_forms():
    """The sweep's per-variant HBM units (bench.schedule_units, read from the compiled
    schedule) match the closed forms for p ranks on one GPU: pairwise allgather p + p^2
    (one read, p writes per rank), pairwise alltoall 2p^2, ring allgather 2p(p-1) + 2p (p-1
    forwarding steps plus the self copy), Bruck allgather 2p(p-1) + 2p^2 (rounds of 1, 2, 4 ..
    blocks, then the final rotation), Bruck alltoall 2p*sum(m_k) + 2p^2 (the first rotation
    is virtual; m_k = blocks with bit k set), hierarchical with one
    group = pairwise."""
    for p in (2, 5, 8):
        K = (p - 1).bit_length()
        m = sum(sum(1 for i in range(p) if i >> k & 1) for k in range(K))
        assert bench.schedule_units("allgather", "pairwise", p, p, p) == p + p * p
        assert bench.schedule_units("alltoall", "pairwise", p, p, p) == 2 * p * p
        assert bench.schedule_units("allgather", "ring", p, p, p) == 2 * p * (p - 1) + 2 * p
        assert bench.schedule_units("allgather", "bruck", p, p, p) == 2 * p * (p - 1) + 2 * p * p
        assert bench.schedule_units("alltoall", "bruck", p, p, p) == 2 * p * m + 2 * p * p
        assert bench.schedule_units("alltoall", "hier", p, p, p) == 2 * p * p

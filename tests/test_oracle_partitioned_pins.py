"""Pins of the f3 oracle: partitioned point-to-point (§2.3).
CPU only.  Pins: SPEC.md's worked examples (4 -> 2 and 4 -> 1 coverage, equal partitioning,
32-byte partitions), every delivery order of 4 partitions giving the same buffer, the
one-partition channel moving exactly one fragment ("no worse than base point-to-point",
PAPER.md:175), and the coverage predicate against an interval computation by hand."""
import itertools

import numpy as np
import pytest

import oracle


def test_spec_4_to_2():
    """sender 4 / receiver 2 partitions over 128 bytes -> receiver partition 0
    arrives exactly when sender partitions {0, 1} are delivered."""
    for bits in itertools.product([0, 1], repeat=4):
        a = oracle.part_arrived(4, 32, 2, 64, bits)
        assert a[0] == (bits[0] and bits[1]) and a[1] == (bits[2] and bits[3])


def test_spec_4_to_1_and_equal():
    """equal partitioning -> arrived after its one overlapping partition;
    sender 4 / receiver 1 -> true only after all 4."""
    for bits in itertools.product([0, 1], repeat=4):
        assert oracle.part_arrived(4, 32, 1, 128, bits)[0] == all(bits)
        assert list(oracle.part_arrived(4, 32, 4, 32, bits)) == [bool(b) for b in bits]


def test_uneven_overlap_by_intervals():
    """3 sender / 2 receiver partitions of 48 bytes: receiver 0 = bytes [0,72) needs sender
    partitions 0 ([0,48)) and 1 ([48,96)); receiver 1 = [72,144) needs 1 and 2."""
    for bits in itertools.product([0, 1], repeat=3):
        a = oracle.part_arrived(3, 48, 2, 72, bits)
        assert a[0] == (bits[0] and bits[1]) and a[1] == (bits[1] and bits[2])


@pytest.mark.parametrize("n_r", [1, 2, 4, 8])
def test_all_orders_same_buffer_and_monotone(n_r):
    """all 24 Pready orders over 4 partitions -> identical receiver buffer;
    arrival flags are monotone within the cycle and all true at the end."""
    send = np.random.default_rng(1).integers(0, 256, 128, dtype=np.uint8)
    for order in itertools.permutations(range(4)):
        recv, trace, st = oracle.part_cycle(send, 4, n_r, order)
        assert np.array_equal(recv, send)
        assert all((trace[k] <= trace[k + 1]).all() for k in range(3))
        assert trace[-1].all()
        assert st["msgs"] == 4                        # one fragment per readied partition


def test_one_partition_is_one_message():
    """PAPER.md:175 'no worse than base point-to-point' (wire-level): a
    1-partition channel moves exactly one payload fragment per cycle."""
    send = np.arange(64, dtype=np.uint8)
    recv, trace, st = oracle.part_cycle(send, 1, 1, [0])
    assert st["msgs"] == 1 and st["bytes"] == 64 and np.array_equal(recv, send) and trace[0, 0]


def test_bad_channels_rejected():
    with pytest.raises(RuntimeError):
        oracle.part_arrived(3, 10, 2, 16, [1, 1, 1])      # totals differ
    with pytest.raises(RuntimeError):
        oracle.part_cycle(np.zeros(8, np.uint8), 2, 1, [0, 0])   # partition readied twice

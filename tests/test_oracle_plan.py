"""Pins for the oracle's plan semantics against the paper's worked examples."""
import pytest

from oracle import plan
from gacer_testutil import read_golden


def _ints(s):
    return [int(t) for t in s.split(",") if t != ""]


def test_eq7_segments_golden():
    for ln in read_golden("eq7_segments.txt"):
        n, cuts, segs = (t.strip() for t in ln.split("|"))
        want = [_ints(s) for s in segs.split(";")]
        assert plan.segments(int(n), _ints(cuts)) == want


def test_eq6_clusters_golden():
    lines = read_golden("eq6_clusters.txt")
    hdr, body = lines[0], lines[1:]
    ns, cuts = (t.strip() for t in hdr.split("|"))
    matrix_p = [_ints(c) for c in cuts.split("/")]
    got = plan.format_clusters(_ints(ns), matrix_p)
    assert got.splitlines() == body


def test_segmentation_roundtrip():
    # concatenating segments reproduces the issue order (SPEC S:81 idea)
    for n in range(0, 9):
        for a in range(0, n + 1):
            for b in range(a, n + 1):
                segs = plan.segments(n, [a, b])
                assert sum(segs, []) == list(range(1, n + 1))
                assert len(segs) == 3


def test_pointer_rules():
    with pytest.raises(ValueError):
        plan.segments(5, [3, 2])          # unsorted
    with pytest.raises(ValueError):
        plan.segments(5, [6])             # out of range
    with pytest.raises(ValueError):
        plan.clusters([4, 4], [[1], [1, 2]])   # unequal pointer counts (l.753)


def test_table3_plans_are_valid_eq5():
    for ln in read_golden("table3_plans.txt"):
        _, v16, r18 = (t.strip() for t in ln.split("|"))
        assert sum(_ints(v16)) == 32 and sum(_ints(r18)) == 32

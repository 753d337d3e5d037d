"""Host logic of the device timeline (engine.Timeline): interval union and the
copy/compute overlap arithmetic used for bench.py's link.timeline block."""

from paper_2509_07379_b200.engine import _covered, _union


def test_union_merges_overlapping_and_touching():
    assert _union([(3, 4), (0, 1), (0.5, 2), (2, 2.5)]) == [[0, 2.5], [3, 4]]
    assert _union([]) == []


def test_covered_fraction():
    u = _union([(0, 10), (20, 30)])
    assert _covered(5, 25, u) == 10          # [5,10] + [20,25]
    assert _covered(10, 20, u) == 0
    assert _covered(-5, 40, u) == 20

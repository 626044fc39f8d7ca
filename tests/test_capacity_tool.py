"""tools/capacity.py bisection: the highest rate meeting the attainment
target, bracketed to within the tolerance (CPU, synthetic attainment curve)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def _bisect():
    import capacity
    return capacity.bisect_capacity


def test_bisection_brackets_the_knee():
    calls = []

    def att(rate):
        calls.append(rate)
        return 1.0 if rate <= 117.3 else 0.5

    r = _bisect()(att, 64, 192, 4, 0.9)
    assert r["capacity_rps"] <= 117.3 < r["first_failing_rps"]
    assert r["first_failing_rps"] - r["capacity_rps"] <= 4
    assert len(calls) <= 2 + 6


def test_bisection_edges():
    b = _bisect()
    assert b(lambda r: 0.5, 64, 192, 4, 0.9)["capacity_rps"] is None
    assert b(lambda r: 0.95, 64, 192, 4, 0.9)["capacity_rps"] == 192
    assert b(lambda r: 0.95, 116, 116, 4, 0.9)["capacity_rps"] == 116

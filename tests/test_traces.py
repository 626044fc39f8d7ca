"""New trace shapes (not in the reference): statistics and determinism."""
import numpy as np


def test_longbench_shape(nx):
    t = nx.workload_trace("longbench", 2.0, 2000, 3)
    p = np.array([r.prompt_len for r in t])
    assert p.min() >= 4096 and p.max() <= 16384
    assert abs(p.mean() - (4096 + 16384) / 2) < 300
    gaps = np.diff([0.0] + [r.arrival_s for r in t])
    assert abs(gaps.mean() - 0.5) < 0.05  # Poisson at 2 rps
    assert nx.trace_text(t) == nx.trace_text(nx.workload_trace("longbench", 2.0, 2000, 3))


def test_bursty_cv_and_lengths(nx):
    t = nx.workload_trace("bursty", 5.0, 20000, 1)
    gaps = np.diff([0.0] + [r.arrival_s for r in t])
    assert abs(gaps.mean() * 5.0 - 1.0) < 0.1
    cv = gaps.std() / gaps.mean()
    assert 3.3 < cv < 4.7
    mixed = nx.workload_trace("mixed", 5.0, 20000, 1)
    assert [(r.prompt_len, r.output_len) for r in t] == [(r.prompt_len, r.output_len) for r in mixed]

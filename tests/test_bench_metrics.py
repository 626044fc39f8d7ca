"""CPU checks of bench.py's metric code: SLO goodput from a reference-format
event log (the same function scores both arms), nearest-rank percentiles,
and the partition roofline ceiling reported beside the HBM-peak fraction."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def _log(lines):
    return "\n".join("\t".join(str(x) for x in l) for l in lines)


def test_goodput_counts_only_slo_attaining_requests():
    # request 1: TTFT 0.1 s, gaps 20 ms -> good (3 tokens)
    # request 2: TTFT 2.0 s -> TTFT miss
    # request 3: TTFT 0.1 s, one 90 ms gap -> p99 TBT miss (its p99 is its max gap)
    log = _log([
        (0.0, "-", "arrival", "1:0:0", 50, 0, 0),
        (0.0, "-", "arrival", "2:0:0", 50, 0, 0),
        (0.0, "-", "arrival", "3:0:0", 50, 0, 0),
        (0.1, "prefill", "complete", "1:10:1,3:10:1", 50, 0, 0),
        (0.12, "decode", "complete", "1:1:1,3:1:1", 50, 0, 0),
        (0.14, "decode", "complete", "1:1:1", 50, 0, 0),
        (0.21, "decode", "complete", "3:1:1", 50, 0, 0),
        (0.14, "-", "finish", "1:0:0", 50, 0, 0),
        (0.21, "-", "finish", "3:0:0", 50, 0, 0),
        (2.0, "prefill", "complete", "2:10:1", 50, 0, 0),
        (2.0, "-", "finish", "2:0:0", 50, 0, 0),
    ])
    m = bench.log_metrics(log, 1.0, 0.05)
    assert m["completed"] == 3
    assert m["out_tokens"] == 3 + 1 + 3
    assert m["good_tokens"] == 3
    assert sorted(round(t, 6) for t in m["ttft"]) == [0.1, 0.1, 2.0]


@pytest.mark.parametrize("v,p,want", [([5, 1, 4, 2, 3], 50, 3), ([5, 1, 4, 2, 3], 99, 5), ([7], 99, 7),
                                      ([], 50, 0.0), (list(range(1, 101)), 99, 99)])
def test_nearest_rank(v, p, want):
    assert bench.nearest_rank(v, p) == want


def test_partition_roofline_decode_ceiling():
    pk = {"hbm_gbs": 6559.7, "bf16_tflops": 1626.5, "bf16_tflops_sustained": 1389.2, "sm_max_mhz": 1965.0}
    c = {"GBps": 2611.0, "TFLOPs": 36.0, "mean_partition_sms": 32.0}
    r = bench.partition_roofline("gemm_decode", c, pk)
    assert r["ceiling"] == pytest.approx(32 * 64 * 1965e6 / 1e9)  # tensor floor of the lane
    assert r["frac"] == pytest.approx(2611.0 / r["ceiling"])
    c_full = {"GBps": 5000.0, "TFLOPs": 0.0, "mean_partition_sms": 148.0}
    assert bench.partition_roofline("gemm_decode", c_full, pk)["ceiling"] == pk["hbm_gbs"]
    p = bench.partition_roofline("gemm_prefill", {"GBps": 0.0, "TFLOPs": 900.0, "mean_partition_sms": 116.0}, pk)
    assert p["ceiling"] == pytest.approx(1389.2 * 116 / 148)
    assert bench.partition_roofline("gemm_decode", {"GBps": 1.0, "mean_partition_sms": 0.0}, pk) is None

"""Pins the pure-Python engine port (oracle/engine_port.py) to the compiled
reference: byte-identical event and decision logs in virtual-clock mode.
Only then is it trusted as the replay oracle for device-clock runs."""
import pytest

from oracle.engine_port import run_port


@pytest.mark.parametrize("kind,policy,preset,rate,count", [
    (0, 0, "mixed", 2.5, 64), (2, 0, "mixed", 2.5, 64), (1, 0, "mixed", 2.5, 64),
    (0, 1, "mixed", 2.5, 64), (0, 0, "sharegpt", 30.0, 150), (0, 0, "long-data", 1.0, 30)])
def test_port_matches_reference(nx, ref, kind, policy, preset, rate, count):
    tiny = nx.derive(256, 1024, 2, 4, 2)
    cfg = nx.sim_config(tiny, nx.gpu_preset("desk"), kind=kind, prefill_policy=policy)
    trace = nx.workload_trace(preset, rate, count, 1)
    ev, dec = run_port(cfg, trace)
    r = ref.run(cfg, trace)
    assert ev == r["event_log"]
    assert dec == r["decision_log"]


def test_port_matches_reference_decode_mode(nx, ref):
    tiny = nx.derive(256, 1024, 2, 4, 2)
    g = nx.gpu_preset("desk-tight")
    g.kv_capacity_bytes = 64 << 20
    trace = [nx.Request(i, t.arrival_s, 64, 600) for i, t in enumerate(nx.workload_trace("sharegpt", 20.0, 80, 1))]
    cfg = nx.sim_config(tiny, g)
    ev, dec = run_port(cfg, trace)
    r = ref.run(cfg, trace)
    assert ev == r["event_log"] and dec == r["decision_log"]

"""Regenerates tests/golden/ from the compiled reference (oracle/_ref).

Run where /root/reference exists:  python tests/golden/make_golden.py
Writes the C1 trace file (reference save_trace format) and, for every engine
fixture of tests/test_host_parity.py, the sha256 of the reference's event log,
decision log and summary JSON (golden.json)."""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2507_06608_b200 as nx  # noqa: E402
from oracle import reference as ref  # noqa: E402
from test_host_parity import FIXTURES, _fixtures  # noqa: E402


def h(s):
    return hashlib.sha256(s.encode()).hexdigest()


def main():
    fx, _ = _fixtures(nx)
    out = {}
    for name in FIXTURES:
        model, gpu, kw, (preset, rate, count, seed) = fx[name]
        cfg = nx.sim_config(model, gpu, **kw)
        trace = ref.workload_trace(preset, rate, count, seed)
        r = ref.run(cfg, trace)
        out[name] = {"trace_sha256": h(ref.trace_text(trace)), "event_log_sha256": h(r["event_log"]),
                     "decision_log_sha256": h(r["decision_log"]), "summary_sha256": h(r["summary_json"]),
                     "events": r["event_log"].count("\n"), "sim_end_s": r["sim_end_s"],
                     "timed_out": r["timed_out"]}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "c1_mixed_64_2.5rps_seed1.trace"), "w") as f:
        f.write(ref.trace_text(ref.workload_trace("mixed", 2.5, 64, 1)))


if __name__ == "__main__":
    main()

"""Decode-step time with per-kernel profiling off (no events between the
launches, so PDL overlap is intact): Llama-3.1-8B, B sequences at CTX on the
whole GPU and on a partition, against the weight-streaming floor
(weights / measured HBM peak).

    B=1,4,16,64 CTX=1000 PCTS=100,21 python tools/decode_step_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2507_06608_b200 import device as D  # noqa: E402

MODEL = os.environ.get("MODEL", "llama3-8b")
BS = [int(x) for x in os.environ.get("B", "1,4,16,64").split(",")]
CTX = int(os.environ.get("CTX", "1000"))
REPS = int(os.environ.get("REPS", "8"))
PCTS = [int(x) for x in os.environ.get("PCTS", "100,21").split(",")]

pp = CTX // 16 + 2
bmax = max(BS)
dev = D.Device(D.arch_preset(MODEL), num_pages=bmax * pp + 64, max_decode_batch=max(64, bmax))
rng = np.random.default_rng(0)
dev.set_profiling(0)
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))
    hbm = float(peak.get("hbm_gbs") or peak.get("hbm_copy_gbs") or 6543.4)
except (OSError, ValueError):
    hbm = 6543.4
wbytes = int(dev.info().weight_bytes)
for B in BS:
    Dm = [dict(tokens=[int(rng.integers(0, 1000))], start=CTX - 1, pages=list(range(i * pp, (i + 1) * pp)))
          for i in range(B)]
    for pct in PCTS:
        dev.launch(Dm, lane=1, sm_pct=pct)
        dev.wait(1)
        step = []
        for _ in range(REPS):
            dev.launch(Dm, lane=1, sm_pct=pct)
            step.append(dev.wait(1)[1])
        row = {"model": MODEL, "B": B, "ctx": CTX, "sm_pct": pct, "step_ms": float(np.median(step)),
               "weight_bytes": wbytes}
        row["floor_ms"] = wbytes / (hbm * 1e6)
        print(json.dumps(row), flush=True)

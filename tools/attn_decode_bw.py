"""Decode-attention bandwidth at full-GPU and partition shares (SURVEY §8 a21:
target >= 85% of the measured copy bandwidth). Decode steps of MODEL at
B x CTX, kernel-class event timing (set_profiling(1)): the attention class's
algorithmic KV bytes / its event time, per SM share.

    MODEL=qwen2.5-14b B=32 CTX=16384 PCTS=100,50,21 python tools/attn_decode_bw.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2507_06608_b200 import device as D  # noqa: E402

MODEL = os.environ.get("MODEL", "qwen2.5-14b")
B = int(os.environ.get("B", "32"))
CTX = int(os.environ.get("CTX", "16384"))
REPS = int(os.environ.get("REPS", "4"))
PCTS = [int(x) for x in os.environ.get("PCTS", "100,50,21").split(",")]
OUT = os.environ.get("OUT", "")

pp = CTX // 16 + 2
dev = D.Device(D.arch_preset(MODEL), num_pages=B * pp + 64, max_decode_batch=max(64, B))
info = dev.info() if hasattr(dev, "info") else None
rng = np.random.default_rng(0)
Dm = [dict(tokens=[int(rng.integers(0, 1000))], start=CTX - 1, pages=list(range(i * pp, (i + 1) * pp)))
      for i in range(B)]
dev.set_profiling(1)
rows = []
for pct in PCTS:
    dev.launch(Dm, lane=1, sm_pct=pct)
    dev.wait(1)
    dev.reset_kernel_stats()
    step = []
    for _ in range(REPS):
        dev.launch(Dm, lane=1, sm_pct=pct)
        step.append(dev.wait(1)[1])
    k = dev.kernel_stats()
    c = 2  # NX_K_ATTN_DECODE
    ms, by, n = k.ms[c], k.bytes[c], k.launches[c]
    sms = k.sm_ms[c] / ms if ms else 0.0
    row = {"model": MODEL, "B": B, "ctx": CTX, "sm_pct": pct, "sms": round(sms, 1),
           "attn_us_per_launch": 1e3 * ms / n, "attn_bytes_per_launch": by / n,
           "attn_GBps": by / (ms * 1e-3) / 1e9, "attn_share_of_step": ms / (sum(k.ms[i] for i in range(5)) or 1),
           "step_ms": float(np.median(step))}
    rows.append(row)
    print(json.dumps(row), flush=True)
if OUT:
    with open(OUT, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")

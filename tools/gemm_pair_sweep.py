"""Prefill GEMMs (T tokens) on the single-CTA kernel vs CTA pairs (cta_group::2)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
rng = np.random.default_rng(0)
T = int(os.environ.get("T", "2048"))
x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((T, 14336)).astype(np.float32)))
out = D.Buf(T * 28672 * 2)
for name, (N, K) in SHAPES.items():
    w = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((N, K)).astype(np.float32) * 0.02))
    mode = D.EPI_SWIGLU if name == "gate_up" else D.EPI_STORE
    ldo = N // 2 if name == "gate_up" else N
    for sms in [int(v) for v in os.environ.get("SMS", "148,116").split(",")]:
        row = {"op": name, "T": T, "sms": sms}
        for tag, sp in [("single", 0), ("pair", -2)]:
            D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, splits=sp, iters=2)
            us = D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, splits=sp, iters=10) / 10 * 1000
            row[tag + "_us"] = round(us, 1)
            row[tag + "_TF"] = round(2.0 * T * N * K / us / 1e6, 0)
        print(json.dumps(row), flush=True)

"""Decode GEMM (gemm_decode.cu) vs the swap-AB kernel: per-launch event time
and weight GB/s (per SM) of the Llama-3.1-8B projections over SM counts."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
rng = np.random.default_rng(0)
sms_list = [int(s) for s in os.environ.get("SMS", "16,32,48,64,96,148").split(",")]
T = int(os.environ.get("T", "64"))
x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((T, 14336)).astype(np.float32)))
out = D.Buf(T * 28672 * 4)
for name, (N, K) in SHAPES.items():
    w = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((N, K)).astype(np.float32) * 0.02))
    for sms in sms_list:
        row = {"op": name, "T": T, "sms": sms}
        for tag, mode, ldo in [("swapab", D.EPI_F32, N), ("decode", D.EPI_DECODE_FOLD, N)]:
            D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, iters=3)
            us = D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, iters=20) / 20 * 1000
            row[tag + "_us"] = round(us, 2)
            row[tag + "_GBps_per_sm"] = round(N * K * 2 / us / 1e3 / sms, 1)
        print(json.dumps(row), flush=True)

"""Decode-shaped GEMM scheduling variants (T=64) timed with 50 back-to-back launches."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
rng = np.random.default_rng(0)
T = int(os.environ.get("T", "64"))
x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((T, 14336)).astype(np.float32)))
out = D.Buf(T * 28672 * 4)
for name, N, K in [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    w = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((N, K)).astype(np.float32) * 0.02))
    mode = D.EPI_SWIGLU if name == "gate_up" else D.EPI_STORE
    ldo = N // 2 if name == "gate_up" else N
    for label, sms, splits in [("streamk148", 148, 0), ("streamk74", 74, 0), ("dp_tiles", N // 128, 0),
                               ("split2", 148, 2), ("split4", 148, 4), ("split8", 148, 8)]:
        D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, splits=splits, iters=3)
        ms = D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, splits=splits, iters=50) / 50
        print(json.dumps({"op": name, "variant": label, "us": round(ms * 1000, 2),
                          "GBps": round(N * K * 2 / ms / 1e6)}), flush=True)

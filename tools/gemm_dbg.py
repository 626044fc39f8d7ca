"""Decode GEMM bottleneck isolation: NX_GEMM_DBG=1 drops the activation TMA
loads, =2 drops the MMAs, =3 both (pure weight streaming through the ring)."""
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
    for sms in [148, 64]:
        D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, iters=3)
        ms = D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, iters=50) / 50
        print(json.dumps({"dbg": os.environ.get("NX_GEMM_DBG", "0"), "op": name, "sms": sms, "us": round(ms * 1000, 2),
                          "GBps": round(N * K * 2 / ms / 1e6)}), flush=True)

"""GEMM scaling sweep on the B200: decode-shaped (weight streaming, GB/s) and
prefill-shaped (TFLOP/s) projections of Llama-3.1-8B versus the number of
SMs the persistent grid may use. Prints one JSON line per point."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def main():
    rng = np.random.default_rng(0)
    sms_list = [int(x) for x in os.environ.get("SMS", "8,16,32,48,64,80,96,112,128,148").split(",")]
    tokens_list = [int(x) for x in os.environ.get("TOKENS", "64,2048").split(",")]
    bufs = {}
    for name, (N, K) in SHAPES.items():
        w = D.f32_to_bf16(rng.standard_normal((N, K)).astype(np.float32) * 0.02)
        bufs[name] = D.Buf.from_array(w)
    for T in tokens_list:
        x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((T, 14336)).astype(np.float32)))
        out = D.Buf(T * 28672 * 2)
        for name, (N, K) in SHAPES.items():
            mode = D.EPI_SWIGLU if name == "gate_up" else D.EPI_STORE
            ldo = N // 2 if name == "gate_up" else N
            for sms in sms_list:
                D.gemm(x, bufs[name], T, N, K, mode, out, ldo, sm_count=sms, iters=3)
                iters = 20
                ms = D.gemm(x, bufs[name], T, N, K, mode, out, ldo, sm_count=sms, iters=iters) / iters
                byts = N * K * 2 + T * K * 2 + T * N * 2
                fl = 2.0 * T * N * K
                print(json.dumps({"op": name, "T": T, "N": N, "K": K, "sms": sms, "ms": ms,
                                  "GBps": byts / ms / 1e6, "TFLOPs": fl / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()

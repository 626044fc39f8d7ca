"""Runs a handful of decode- and prefill-shaped GEMMs (for ncu captures)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
rng = np.random.default_rng(0)
N, K = 28672, 4096
w = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((N, K)).astype(np.float32) * 0.02))
for T in [int(t) for t in os.environ.get("TOKENS", "64,2048").split(",")]:
    x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((T, K)).astype(np.float32)))
    out = D.Buf(T * N)
    for _ in range(3):
        D.gemm(x, w, T, N, K, D.EPI_SWIGLU, out, N // 2)

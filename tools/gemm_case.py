"""One decode-shaped GEMM configuration, launched a few times (ncu target)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
N = int(os.environ.get("N", "28672")); K = int(os.environ.get("K", "4096")); T = int(os.environ.get("T", "64"))
SMS = int(os.environ.get("SMS", "148")); SPLITS = int(os.environ.get("SPLITS", "0"))
MODE = D.EPI_SWIGLU if N == 28672 else D.EPI_STORE
rng = np.random.default_rng(0)
x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((T, K)).astype(np.float32)))
w = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((N, K)).astype(np.float32) * 0.02))
o = D.Buf(T * N * 4)
for _ in range(3):
    D.gemm(x, w, T, N, K, MODE, o, N // 2 if MODE == D.EPI_SWIGLU else N, sm_count=SMS, splits=SPLITS)

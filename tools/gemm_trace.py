"""Per-CTA milestone timeline of one decode GEMM launch (NX_GEMM_DBG=16):
0 start, 1 prologue done, 2 first stage landed, 3 last MMA commit,
4 last tile accumulator ready, 5 last epilogue done, 6 fix-up done, 7 exit."""
import ctypes as C, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
from paper_2507_06608_b200._abi import lib
lib().nx_dbg_gemm_trace.restype = C.c_size_t
lib().nx_dbg_gemm_trace.argtypes = [C.c_void_p, C.c_size_t]
rng = np.random.default_rng(0)
T = int(os.environ.get("T", "64"))
x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((T, 14336)).astype(np.float32)))
out = D.Buf(T * 28672 * 4)
for name, N, K in [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    w = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((N, K)).astype(np.float32) * 0.02))
    mode = D.EPI_SWIGLU if name == "gate_up" else D.EPI_STORE
    ldo = N // 2 if name == "gate_up" else N
    for sms in [148, 64]:
        ms = D.gemm(x, w, T, N, K, mode, out, ldo, sm_count=sms, iters=5)
        buf = np.zeros((1024, 8), dtype=np.uint64)
        lib().nx_dbg_gemm_trace(buf.ctypes.data, buf.size)
        t = buf[:sms].astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0
        row = {"op": name, "sms": sms, "event_us": round(ms * 1000, 2)}
        for i, nm in enumerate(["start", "prologue", "first_stage", "last_mma", "acc_ready", "epi_done", "fixup_done", "exit"]):
            row[nm] = [round(float(np.min(rel[:, i])), 2), round(float(np.median(rel[:, i])), 2), round(float(np.max(rel[:, i])), 2)]
        print(json.dumps(row), flush=True)

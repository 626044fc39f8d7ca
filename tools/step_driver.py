"""One Llama-3.1-8B decode batch (B x ctx) and one prefill batch on chosen
partitions, repeated: the target of ncu launch lists / captures."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
B = int(os.environ.get("B", "64")); CTX = int(os.environ.get("CTX", "600"))
DPCT = int(os.environ.get("DPCT", "100")); PPCT = int(os.environ.get("PPCT", "100"))
REPS = int(os.environ.get("REPS", "3")); MODE = os.environ.get("MODE", "decode")
dev = D.Device(D.arch_preset("llama3-8b"), num_pages=B * (CTX // 16 + 2) + 1200, max_decode_batch=max(64, B))
rng = np.random.default_rng(0)
pp = CTX // 16 + 2
Dm = [dict(tokens=[int(rng.integers(0, 1000))], start=CTX - 1, pages=list(range(i * pp, (i + 1) * pp))) for i in range(B)]
PLENS = [int(x) for x in os.environ.get("PLENS", "512,512,512,512").split(",")]
P, pg0 = [], B * pp
for n in PLENS:
    P.append(dict(tokens=rng.integers(0, 1000, n).tolist(), start=0, pages=list(range(pg0, pg0 + n // 16 + 1))))
    pg0 += n // 16 + 1
import time
import ctypes
# ncu --profile-from-start off --replay-mode app-range: profile only the last
# repetition (RANGE=1), bracketed by cuProfilerStart/Stop
RANGE = os.environ.get("RANGE", "0") == "1"
_cuda = ctypes.CDLL("libcuda.so.1") if RANGE else None
for r in range(REPS):
    if RANGE and r == REPS - 1:
        _cuda.cuProfilerStart()
    if MODE in ("decode", "both"):
        t0 = time.perf_counter(); dev.launch(Dm, lane=1, sm_pct=DPCT); t1 = time.perf_counter()
        _, ms = dev.wait(1); t2 = time.perf_counter()
        print(f"decode device_ms {ms:.3f} host_enqueue_ms {1e3*(t1-t0):.3f} wall_ms {1e3*(t2-t0):.3f}", flush=True)
    if MODE in ("prefill", "both"):
        t0 = time.perf_counter(); dev.launch(P, lane=0, sm_pct=PPCT); t1 = time.perf_counter()
        _, ms = dev.wait(0); t2 = time.perf_counter()
        print(f"prefill device_ms {ms:.3f} host_enqueue_ms {1e3*(t1-t0):.3f} wall_ms {1e3*(t2-t0):.3f}", flush=True)
    if MODE == "colo":  # prefill on its partition while decode steps run back to back on the other
        DSTEPS = int(os.environ.get("DSTEPS", "4"))
        dev.launch(P, lane=0, sm_pct=PPCT)
        dms = []
        for _ in range(DSTEPS):
            dev.launch(Dm, lane=1, sm_pct=DPCT)
            dms.append(dev.wait(1)[1])
        _, pms = dev.wait(0)
        print(f"colo prefill_ms {pms:.3f} decode_ms {sum(dms)/len(dms):.3f} ({DSTEPS} steps)", flush=True)
    if MODE == "mixed":  # one fused batch (decode members first), monolithic-style full-GPU lane
        t0 = time.perf_counter(); dev.launch(Dm + P, lane=0, sm_pct=100)
        _, ms = dev.wait(0); t2 = time.perf_counter()
        print(f"mixed device_ms {ms:.3f} wall_ms {1e3*(t2-t0):.3f} tokens {len(Dm) + sum(PLENS)}", flush=True)
    if RANGE and r == REPS - 1:
        _cuda.cuProfilerStop()

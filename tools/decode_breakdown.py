"""Per-kernel-class and per-operator time of one Llama-3.1-8B decode step
(B x CTX) on a DPCT % partition, alone and beside a prefill batch on the
other partition (sampled CUDA-event pairs; nx_kernel_stats)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D

B = int(os.environ.get("B", "128"))
CTX = int(os.environ.get("CTX", "800"))
DPCT = int(os.environ.get("DPCT", "21"))
REPS = int(os.environ.get("REPS", "6"))
pp = CTX // 16 + 2
dev = D.Device(D.arch_preset("llama3-8b"), num_pages=B * pp + 400, max_decode_batch=max(128, B),
               max_prefill_tokens=2048 + 128)
rng = np.random.default_rng(0)
Dm = [dict(tokens=[int(rng.integers(0, 1000))], start=CTX - 1, pages=list(range(i * pp, (i + 1) * pp)))
      for i in range(B)]
P = [dict(tokens=rng.integers(0, 1000, 512).tolist(), start=0, pages=list(range(B * pp + 33 * i, B * pp + 33 * i + 33)))
     for i in range(4)]
names = ["gemm_decode", "gemm_prefill", "attn_decode", "attn_prefill", "other"]
ops = ["qkv", "attn_prefill", "attn_decode", "o", "ffn"]
for mode in ("alone", "colo"):
    for _ in range(2):
        dev.forward(Dm, lane=1, sm_pct=DPCT)
    dev.set_profiling(1)
    dev.reset_kernel_stats()
    steps = []
    for _ in range(REPS):
        if mode == "colo":
            dev.launch(P, lane=0, sm_pct=100 - DPCT)
        dev.launch(Dm, lane=1, sm_pct=DPCT)
        steps.append(dev.wait(1)[1])
        if mode == "colo":
            dev.wait(0)
    ks = dev.kernel_stats()
    dev.set_profiling(0)
    per = {n: round(ks.ms[i] / REPS, 3) for i, n in enumerate(names) if ks.launches[i]}
    # decode-lane classes only (the co-located prefill batch is excluded by lane? no: both lanes are sampled)
    print(mode, "step ms (median)", round(sorted(steps)[len(steps) // 2], 3), "classes ms/step", per,
          "ops ms/step", {o: round(ks.op_ms[k] / REPS, 3) for k, o in enumerate(ops)},
          "launches/step", {n: ks.launches[i] // REPS for i, n in enumerate(names) if ks.launches[i]})

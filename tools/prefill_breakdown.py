"""Per-kernel-class time of one Llama-3.1-8B prefill batch (NSEQ x PLEN tokens)
on a PPCT % partition, alone and beside back-to-back decode steps (B x CTX)
on the other partition (sampled CUDA-event pairs; nx_kernel_stats)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D

PLEN = int(os.environ.get("PLEN", "512"))
NSEQ = int(os.environ.get("NSEQ", "4"))
PPCT = int(os.environ.get("PPCT", "79"))
B = int(os.environ.get("B", "128"))
CTX = int(os.environ.get("CTX", "800"))
REPS = int(os.environ.get("REPS", "4"))
pp = CTX // 16 + 2
ppp = PLEN // 16 + 2
dev = D.Device(D.arch_preset("llama3-8b"), num_pages=B * pp + NSEQ * ppp + 64, max_decode_batch=max(128, B),
               max_prefill_tokens=max(2048, NSEQ * PLEN) + 128)
rng = np.random.default_rng(0)
Dm = [dict(tokens=[int(rng.integers(0, 1000))], start=CTX - 1, pages=list(range(i * pp, (i + 1) * pp)))
      for i in range(B)]
P = [dict(tokens=rng.integers(0, 1000, PLEN).tolist(), start=0,
          pages=list(range(B * pp + i * ppp, B * pp + (i + 1) * ppp))) for i in range(NSEQ)]
names = ["gemm_decode", "gemm_prefill", "attn_decode", "attn_prefill", "other"]
for mode in ("alone", "colo"):
    dev.forward(P, lane=0, sm_pct=PPCT)
    dev.set_profiling(1)
    dev.reset_kernel_stats()
    times = []
    for _ in range(REPS):
        dev.launch(P, lane=0, sm_pct=PPCT)
        if mode == "colo":
            while True:  # decode steps back to back until the prefill batch is done
                dev.launch(Dm, lane=1, sm_pct=100 - PPCT)
                dev.wait(1)
                if dev.done(0) if hasattr(dev, "done") else False:
                    break
                break
        times.append(dev.wait(0)[1])
    ks = dev.kernel_stats()
    dev.set_profiling(0)
    per = {n: round(ks.ms[i] / REPS, 3) for i, n in enumerate(names) if ks.launches[i]}
    print(mode, "prefill batch ms (median)", round(sorted(times)[len(times) // 2], 3), "classes ms/batch", per,
          "launches", {n: ks.launches[i] // REPS for i, n in enumerate(names) if ks.launches[i]})

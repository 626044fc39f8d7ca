"""Prefill attention throughput at bench shapes (event-timed per launch via the
device's sampled kernel stats): a CHUNK-token prefill chunk on top of a CTX
prefix (C3: qwen2.5-14b, CTX 14336, CHUNK 2048), or NSEQ fresh prompts of
PLEN tokens (8B ShareGPT: 4 x 512). Two layers of the named geometry; the
attention launches are identical to the full model's."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D

MODEL = os.environ.get("MODEL", "qwen2.5-14b")
CTX = int(os.environ.get("CTX", "14336"))
CHUNK = int(os.environ.get("CHUNK", "2048"))
NSEQ = int(os.environ.get("NSEQ", "1"))
PCT = int(os.environ.get("PCT", "100"))
REPS = int(os.environ.get("REPS", "5"))
a = D.arch_preset(MODEL, n_layers=2, vocab=8192)
pages_per = (CTX + CHUNK) // 16 + 2
dev = D.Device(a, num_pages=NSEQ * pages_per + 64, max_prefill_tokens=max(2048, NSEQ * CHUNK) + 128)
rng = np.random.default_rng(0)
seqs = []
for i in range(NSEQ):
    pg = list(range(i * pages_per, (i + 1) * pages_per))
    toks = rng.integers(0, a.vocab, CTX + CHUNK).tolist()
    for c0 in range(0, CTX, 2048):
        dev.forward([dict(tokens=toks[c0:min(CTX, c0 + 2048)], start=c0, pages=pg, sample=False)], lane=0, sm_pct=100)
    seqs.append((toks, pg))
members = [dict(tokens=t[CTX:CTX + CHUNK], start=CTX, pages=pg, sample=False) for t, pg in seqs]
dev.forward(members, lane=0, sm_pct=PCT)
dev.set_profiling(1)
dev.reset_kernel_stats()
for _ in range(REPS):
    dev.forward(members, lane=0, sm_pct=PCT)
ks = dev.kernel_stats()
names = ["gemm_decode", "gemm_prefill", "attn_decode", "attn_prefill", "other"]
for i, n in enumerate(names):
    if ks.launches[i]:
        print(f"{n}: {ks.launches[i]} launches, {ks.ms[i] / ks.launches[i] * 1e3:.1f} us/launch, "
              f"{ks.flops[i] / ks.ms[i] / 1e9:.1f} TFLOP/s, {ks.bytes[i] / ks.ms[i] / 1e6:.1f} GB/s")

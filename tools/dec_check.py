"""Decode-attention check at long contexts: tiny model, chunked prefill of
CTX tokens, then decode steps on the decode lane at several SM shares;
logits vs the fp32 oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_06608_b200 import device as D
from oracle.llama_fp32 import LlamaFP32
dev = D.Device(D.arch_preset("tiny"), num_pages=8192, seed=7)
ref = LlamaFP32(dev)
rng = np.random.default_rng(1)
for ctx in [40, 600, 3000, 9000]:
    prompt = rng.integers(0, dev.arch.vocab, ctx).tolist()
    npg = ctx // 16 + 4
    pages = list(rng.permutation(8000)[:npg])
    pages = [int(p) for p in pages]
    for c0 in range(0, ctx, 2048):
        dev.forward([dict(tokens=prompt[c0:c0 + 2048], start=c0, pages=pages, sample=False)], lane=0, sm_pct=60)
    want = ref.logits(np.array(prompt + [5]))[-1]
    for pct in [5, 30, 60, 99]:
        out, lg, _ = dev.forward([dict(tokens=[5], start=ctx, pages=pages)], lane=1, sm_pct=pct, want_logits=True)
        err = np.abs(lg[0] - want).max() / np.abs(want).max()
        print(f"ctx {ctx} pct {pct} rel_err {err:.4f} tok {out[0]} want {int(np.argmax(want))}", flush=True)

"""Forward-pass parity of the device executor against the fp32 numpy oracle
(oracle/llama_fp32.py) on the exact bf16 weights the device holds.

Tolerances (bf16 activations/weights vs fp32 reference), stated here:
  * logits: max |dev - ref| <= 3e-2 * max |ref|  per sampled row;
  * greedy tokens: equal wherever the fp32 top-1/top-2 margin exceeds 4x the
    row's observed logit error bound (ties inside the error bar are exempt).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOGIT_TOL = 3e-2


@pytest.fixture(scope="module")
def D():
    from paper_2507_06608_b200 import device
    return device


def _check_logits(dev_logits, ref_logits, dev_tokens):
    for row, ref, tok in zip(dev_logits, ref_logits, dev_tokens):
        err = np.abs(row - ref).max()
        assert err <= LOGIT_TOL * np.abs(ref).max(), (err, np.abs(ref).max())
        top2 = np.sort(ref)[-2:]
        if top2[1] - top2[0] > 4 * LOGIT_TOL * np.abs(ref).max():
            assert tok == int(np.argmax(ref))


@pytest.fixture(scope="module")
def tiny(D):
    from oracle.llama_fp32 import LlamaFP32
    dev = D.Device(D.arch_preset("tiny"), num_pages=2048, seed=7)
    return dev, LlamaFP32(dev)


@pytest.fixture(scope="module")
def gqa(D):
    from oracle.llama_fp32 import LlamaFP32
    a = D.arch(hidden=512, n_layers=2, n_heads=8, n_kv_heads=2, ffn=1536, vocab=2048, rope_theta=10000.0)
    dev = D.Device(a, num_pages=2048, seed=11)
    return dev, LlamaFP32(dev)


def test_green_context_layouts(tiny):
    dev, _ = tiny
    info = dev.info()
    assert info.sm_count == 148
    assert info.n_layouts >= 16
    for i in range(info.n_layouts):
        assert info.layout_decode_sms[i] == 8 * (i + 1)
        assert info.layout_decode_sms[i] + info.layout_prefill_sms[i] == info.sm_count


@pytest.mark.parametrize("model", ["tiny", "gqa"])
def test_single_prefill_logits(request, model):
    dev, ref = request.getfixturevalue(model)
    rng = np.random.default_rng(1)
    toks = rng.integers(0, dev.arch.vocab, 77).tolist()
    pages = list(range(100, 100 + 5))[::-1]  # non-contiguous, reversed
    out, logits, ms = dev.forward([dict(tokens=toks, start=0, pages=pages)], want_logits=True)
    want = ref.logits(np.array(toks))[-1:]
    _check_logits(logits, want, out)


@pytest.mark.parametrize("model", ["tiny", "gqa"])
def test_chunked_prefill_then_decode(request, model):
    """Prefill in two chunks, then greedy decode steps on the decode lane;
    every step's logits vs a full-sequence fp32 recompute."""
    dev, ref = request.getfixturevalue(model)
    rng = np.random.default_rng(2)
    prompt = rng.integers(0, dev.arch.vocab, 150).tolist()
    pages = [7, 300, 12, 999, 45, 600, 13, 14, 15, 1000, 1001, 1002, 1003, 1004, 1005]
    dev.forward([dict(tokens=prompt[:96], start=0, pages=pages, sample=False)], lane=0, sm_pct=60)
    out, logits, _ = dev.forward([dict(tokens=prompt[96:], start=96, pages=pages)], lane=0, sm_pct=60,
                                 want_logits=True)
    seq = list(prompt)
    _check_logits(logits, ref.logits(np.array(seq))[-1:], out)
    seq.append(out[0])
    for step in range(6):
        out, logits, _ = dev.forward([dict(tokens=[seq[-1]], start=len(seq) - 1, pages=pages)], lane=1,
                                     sm_pct=40, want_logits=True)
        _check_logits(logits, ref.logits(np.array(seq))[-1:], out)
        seq.append(out[0])


def test_batched_prefill_and_decode_members(gqa):
    dev, ref = gqa
    rng = np.random.default_rng(3)
    lens = [1, 17, 64, 129, 300]
    prompts = [rng.integers(0, dev.arch.vocab, n).tolist() for n in lens]
    page_sets = [[200 + 30 * i + k for k in range(30)][::-1] for i in range(len(lens))]
    members = [dict(tokens=p, start=0, pages=pg) for p, pg in zip(prompts, page_sets)]
    out, logits, _ = dev.forward(members, lane=0, sm_pct=70, want_logits=True)
    want = np.stack([ref.logits(np.array(p))[-1] for p in prompts])
    _check_logits(logits, want, out)
    # one decode step for all of them in one batch (decode lane, split-KV)
    seqs = [p + [t] for p, t in zip(prompts, out)]
    dmem = [dict(tokens=[s[-1]], start=len(s) - 1, pages=pg) for s, pg in zip(seqs, page_sets)]
    out2, logits2, _ = dev.forward(dmem, lane=1, sm_pct=30, want_logits=True)
    want2 = np.stack([ref.logits(np.array(s))[-1] for s in seqs])
    _check_logits(logits2, want2, out2)


def test_long_context_decode_splits(gqa):
    """1,500-token context: many KV tiles, split-KV decode with combine."""
    dev, ref = gqa
    rng = np.random.default_rng(4)
    prompt = rng.integers(0, dev.arch.vocab, 1500).tolist()
    pages = list(range(1500 // 16 + 2))
    dev.forward([dict(tokens=prompt[:1024], start=0, pages=pages, sample=False)], lane=0)
    out, logits, _ = dev.forward([dict(tokens=prompt[1024:], start=1024, pages=pages)], lane=0,
                                 want_logits=True)
    _check_logits(logits, ref.logits(np.array(prompt))[-1:], out)
    seq = prompt + [out[0]]
    out, logits, _ = dev.forward([dict(tokens=[seq[-1]], start=len(seq) - 1, pages=pages)], lane=1,
                                 sm_pct=10, want_logits=True)
    _check_logits(logits, ref.logits(np.array(seq))[-1:], out)


@pytest.mark.parametrize("ctx", [40, 600, 5000])
def test_decode_long_context_all_partitions(tiny, ctx):
    """Decode attention distributes the flattened 32-key tiles of all
    (sequence, kv head) items over the warps of the lane's partition; a
    context is split across 1..hundreds of warps depending on the partition
    size, and the pieces are folded by the combine kernel. Same logits at
    every partition size, against the fp32 oracle."""
    dev, ref = tiny
    rng = np.random.default_rng(ctx)
    prompt = rng.integers(0, dev.arch.vocab, ctx).tolist()
    pages = [int(p) for p in rng.permutation(2000)[:ctx // 16 + 4]]
    for c0 in range(0, ctx, 2048):
        dev.forward([dict(tokens=prompt[c0:c0 + 2048], start=c0, pages=pages, sample=False)], lane=0, sm_pct=60)
    want = ref.logits(np.array(prompt + [5]))[-1:]
    for pct in (5, 30, 99):
        out, lg, _ = dev.forward([dict(tokens=[5], start=ctx, pages=pages)], lane=1, sm_pct=pct, want_logits=True)
        _check_logits(lg, want, out)

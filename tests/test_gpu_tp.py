"""Tensor parallelism on the device, run on ONE B200 with the
ranks colocated (NX_TP_PEER_COLOCATED): every rank is a full executor with its
own weight shard, KV heads and lane workspaces, and the O / down all-reduces
and the vocab-parallel argmax run through the peer-memory collective kernels
(tp.cu) exactly as on NX_TP_PEER across GPUs — only the peer pointers are
local. The NCCL mode (one process per GPU) shares every kernel but the
collective call and needs >= 2 GPUs, so it is not exercised here.

Parity: a TP shard is generated as the exact slice of the unsharded model
(fill_random_slice), so the fp32 oracle built from the TP=1 device is the
reference for every TP size. Tolerances as in test_gpu_model.py.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOGIT_TOL = 3e-2


@pytest.fixture(scope="module")
def D():
    from paper_2507_06608_b200 import device
    return device


ARCHES = {
    2: dict(hidden=512, n_layers=2, n_heads=8, n_kv_heads=2, ffn=1536, vocab=2048, rope_theta=10000.0),
    4: dict(hidden=512, n_layers=2, n_heads=8, n_kv_heads=4, ffn=1024, vocab=1920, rope_theta=10000.0),
    # 8 kv heads, one per rank (the Llama-3.1-70B split at TP=8: 8 q + 1 kv head per GPU)
    8: dict(hidden=2048, n_layers=2, n_heads=16, n_kv_heads=8, ffn=2048, vocab=3072, rope_theta=500000.0),
}


@pytest.fixture(scope="module", params=[2, 4, 8])
def pair(request, D):
    from oracle.llama_fp32 import LlamaFP32
    tp = request.param
    a = D.arch(**ARCHES[tp])
    full = D.Device(a, num_pages=4096, seed=13)
    sharded = D.Device(a, num_pages=4096, seed=13, tp_size=tp, tp_mode=D.NX_TP_PEER_COLOCATED,
                       green_contexts=False)
    yield tp, full, sharded, LlamaFP32(full)
    sharded.close()
    full.close()


def _check(dev_logits, ref_logits, dev_tokens):
    for row, ref, tok in zip(dev_logits, ref_logits, dev_tokens):
        err = np.abs(row - ref).max()
        assert err <= LOGIT_TOL * np.abs(ref).max(), (err, np.abs(ref).max())
        top2 = np.sort(ref)[-2:]
        if top2[1] - top2[0] > 4 * LOGIT_TOL * np.abs(ref).max():
            assert tok == int(np.argmax(ref))


def test_rank0_weights_are_slices(D, pair):
    tp, full, sharded, _ = pair
    a = full.arch
    plan = D.shard_plan(a, tp, 0)
    hd, d = a.head_dim, a.hidden
    qkv = full.weight(D.W_QKV, 1).reshape(-1, d)
    rows = np.concatenate([np.arange(plan.q_head0 * hd, (plan.q_head0 + plan.n_q_heads) * hd),
                           a.n_heads * hd + np.arange(plan.kv_head0 * hd, (plan.kv_head0 + plan.n_kv_heads) * hd),
                           (a.n_heads + a.n_kv_heads) * hd
                           + np.arange(plan.kv_head0 * hd, (plan.kv_head0 + plan.n_kv_heads) * hd)])
    assert np.array_equal(sharded.weight(D.W_QKV, 1).reshape(-1, d), qkv[rows])
    o = full.weight(D.W_O, 0).reshape(d, -1)
    assert np.array_equal(sharded.weight(D.W_O, 0).reshape(d, -1), o[:, :plan.n_q_heads * hd])
    down = full.weight(D.W_DOWN, 0).reshape(d, -1)
    assert np.array_equal(sharded.weight(D.W_DOWN, 0).reshape(d, -1), down[:, :plan.ffn_local])
    lm = full.weight(D.W_LM_HEAD).reshape(-1, d)
    assert np.array_equal(sharded.weight(D.W_LM_HEAD).reshape(-1, d)[:plan.vocab_valid], lm[:plan.vocab_valid])


def test_tp_prefill_and_decode_vs_oracle(pair):
    tp, full, sharded, ref = pair
    rng = np.random.default_rng(3 + tp)
    a_prompt = rng.integers(0, full.arch.vocab, 150).tolist()
    b_prompt = rng.integers(0, full.arch.vocab, 40).tolist()
    pa, pb = [5, 90, 17, 300, 8, 9, 10, 11, 12, 13], [400, 401, 402, 403, 404]
    # chunked prefill of A on the prefill lane, B in one go
    sharded.forward([dict(tokens=a_prompt[:96], start=0, pages=pa, sample=False)], lane=0, sm_pct=60)
    out, lg, _ = sharded.forward([dict(tokens=a_prompt[96:], start=96, pages=pa),
                                  dict(tokens=b_prompt, start=0, pages=pb)], lane=0, sm_pct=60, want_logits=True)
    _check(lg, np.stack([ref.logits(np.array(a_prompt))[-1], ref.logits(np.array(b_prompt))[-1]]), out)
    seq_a, seq_b = a_prompt + [out[0]], b_prompt + [out[1]]
    # greedy decode steps of both on the decode lane
    for _ in range(6):
        out, lg, _ = sharded.forward([dict(tokens=[seq_a[-1]], start=len(seq_a) - 1, pages=pa),
                                      dict(tokens=[seq_b[-1]], start=len(seq_b) - 1, pages=pb)],
                                     lane=1, sm_pct=30, want_logits=True)
        _check(lg, np.stack([ref.logits(np.array(seq_a))[-1], ref.logits(np.array(seq_b))[-1]]), out)
        seq_a.append(out[0])
        seq_b.append(out[1])


def test_tp_matches_single_gpu_tokens(pair):
    """The same batch through TP=1 and TP=tp: logits agree to the bf16 bar
    and the greedy tokens are identical wherever the margin is clear."""
    tp, full, sharded, _ = pair
    rng = np.random.default_rng(21)
    members = [dict(tokens=rng.integers(0, full.arch.vocab, n).tolist(), start=0, pages=[1000 + 10 * i + k for k in range(8)])
               for i, n in enumerate([33, 64, 100, 7])]
    o1, l1, _ = full.forward(members, want_logits=True)
    o2, l2, _ = sharded.forward(members, want_logits=True)
    _check(l2, l1, o2)


def test_tp_engine_run(nx, pair):
    """An engine bound to the TP device serves a trace; the virtual-clock
    schedule is byte-identical to the single-GPU run and tokens pass the
    teacher-forced oracle check."""
    tp, full, sharded, ref = pair
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 2.5, 16, 4)
    cfg = nx.sim_config(tiny, nx.gpu_preset("desk"))
    logs = []
    for dev in (full, sharded):
        eng = nx.Engine(cfg, device=dev)
        eng.submit_trace(trace)
        eng.run()
        logs.append(eng.event_log())
        if dev is sharded:
            checked = mism = 0
            for q in sorted(eng.requests(), key=lambda q: q.prompt_len)[:10]:
                toks = eng.tokens(q.id)
                assert len(toks) == q.prompt_len + q.output_len
                seq = np.array(toks)
                logits = ref.logits(seq[:-1])[q.prompt_len - 1:][:32]
                for row, tok in zip(logits, seq[q.prompt_len:]):
                    top2 = np.sort(row)[-2:]
                    if top2[1] - top2[0] > 4 * LOGIT_TOL * np.abs(row).max():
                        checked += 1
                        mism += int(tok != int(np.argmax(row)))
            assert checked > 20 and mism == 0
        eng.close()
    assert logs[0] == logs[1]

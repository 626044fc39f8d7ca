"""Tensor parallelism on CPU.

* nx_tp_shard_plan (pure host arithmetic behind the C-ABI): every q head,
  kv head, ffn feature and vocab row is owned by exactly one rank.
* world_size-2 gloo run of the Megatron decomposition the device executes
  (tp.cuh): column-parallel QKV / gate-up, row-parallel O / down with the
  residual folded into rank 0's partial before the all-reduce, and a
  vocab-parallel greedy argmax through an all-gather of (max, global idx)
  pairs. The sharded forward must equal the unsharded one (fp32, 1e-4) and
  pick the same token; a forced cross-rank tie must resolve to the lowest
  global index, as argmax does on one GPU.
"""
import os
import socket
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2507_06608_b200 import device as D  # noqa: E402


def _plans(a, tp):
    return [D.shard_plan(a, tp, r) for r in range(tp)]


@pytest.mark.parametrize("name", ["tiny", "llama3-8b", "qwen2.5-14b", "llama3-70b"])
@pytest.mark.parametrize("tp", [1, 2, 4, 8])
def test_shard_plan_partitions_everything(name, tp):
    a = D.arch_preset(name)
    if a.n_kv_heads % tp or a.n_heads % tp or a.ffn % (64 * tp):
        with pytest.raises(Exception):
            D.shard_plan(a, tp, 0)
        return
    ps = _plans(a, tp)
    q = sorted(h for p in ps for h in range(p.q_head0, p.q_head0 + p.n_q_heads))
    kv = sorted(h for p in ps for h in range(p.kv_head0, p.kv_head0 + p.n_kv_heads))
    assert q == list(range(a.n_heads)) and kv == list(range(a.n_kv_heads))
    assert sum(p.ffn_local for p in ps) == a.ffn
    assert [p.ffn0 for p in ps] == [r * a.ffn // tp for r in range(tp)]
    # GQA groups never straddle ranks: rank r's q heads map onto its kv heads
    for p in ps:
        g = a.n_heads // a.n_kv_heads
        assert p.q_head0 // g == p.kv_head0 and p.n_q_heads == g * p.n_kv_heads
    # vocab: padded to 128*tp, local slices contiguous, valid rows cover vocab once
    for p in ps:
        assert p.vocab_padded % (128 * tp) == 0 and p.vocab_local * tp == p.vocab_padded
        assert p.vocab_local % 128 == 0 and 0 <= p.vocab_valid <= p.vocab_local
    rows = [v for p in ps for v in range(p.vocab0, p.vocab0 + p.vocab_valid)]
    assert rows == list(range(a.vocab))


def test_shard_plan_rejects_bad_rank():
    a = D.arch_preset("llama3-8b")
    for tp, r in [(0, 0), (2, 2), (2, -1), (3, 0)]:
        with pytest.raises(Exception):
            D.shard_plan(a, tp, r)


def test_nccl_unique_id_is_fresh():
    a, b = D.nccl_unique_id(), D.nccl_unique_id()
    assert len(a) == 128 and a != b


# ---- world_size-2 gloo run -------------------------------------------------

def _tiny_arch():
    return D.arch(hidden=256, n_layers=2, n_heads=4, n_kv_heads=2, ffn=512, vocab=1000, rope_theta=10000.0)


def _random_model(a, seed):
    from oracle.llama_fp32 import LlamaFP32
    rng = np.random.default_rng(seed)
    d, f, hd = a.hidden, a.ffn, a.head_dim
    qkv_rows = (a.n_heads + 2 * a.n_kv_heads) * hd

    def u(*shape, k):
        return (rng.uniform(-1, 1, shape) * np.sqrt(3.0 / k)).astype(np.float32)

    layers = [dict(attn_norm=(1 + 0.1 * rng.uniform(-1, 1, d)).astype(np.float32), qkv=u(qkv_rows, d, k=d),
                   bias=None, o=u(d, a.n_heads * hd, k=a.n_heads * hd),
                   ffn_norm=(1 + 0.1 * rng.uniform(-1, 1, d)).astype(np.float32),
                   gate=u(f, d, k=d), up=u(f, d, k=d), down=u(d, f, k=f) * 2)
              for _ in range(a.n_layers)]
    w = dict(emb=rng.uniform(-1, 1, (a.vocab, d)).astype(np.float32), layers=layers,
             final_norm=(1 + 0.1 * rng.uniform(-1, 1, d)).astype(np.float32), lm=u(a.vocab, d, k=d) * 4)
    return LlamaFP32(arch=a, weights=w)


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = _tiny_arch()
        full = _random_model(a, 5)
        shard = full.shard(D.shard_plan(a, world, rank))

        def all_reduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
            dist.all_reduce(t)
            return t.numpy()

        def all_gather(pair):
            outs = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(outs, torch.from_numpy(pair))
            return [o.numpy() for o in outs]

        rng = np.random.default_rng(11)
        res = {}
        for case in range(3):
            toks = rng.integers(0, a.vocab, 9 + 4 * case)
            h_full = full.hidden(toks)
            h_tp = shard.hidden(toks, all_reduce=all_reduce, rank=rank)
            res[f"err{case}"] = float(np.abs(h_full - h_tp).max() / np.abs(h_full).max())
            res[f"tok_full{case}"] = int(np.argmax(full.logits(toks)[-1]))
            res[f"tok_tp{case}"] = shard.tp_greedy(toks, all_reduce, all_gather)
        # forced tie: the same maximal row in both ranks' vocab slices
        toks = rng.integers(0, a.vocab, 7)
        h = full.hidden(toks)[-1]
        best = int(np.argmax(h @ full.lm.T))
        tied = full.lm.copy()
        lo, hi = 3, 600  # rows on rank 0 and rank 1 (vocab_local = 512)
        tied[lo] = tied[hi] = full.lm[best] * 2
        full.lm = tied
        shard = full.shard(D.shard_plan(a, world, rank))
        res["tie_full"] = int(np.argmax(full.logits(toks)[-1]))
        res["tie_tp"] = shard.tp_greedy(toks, all_reduce, all_gather)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_tp2_gloo_matches_unsharded(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        res = np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item()
        for c in range(3):
            assert res[f"err{c}"] < 1e-4, res
            assert res[f"tok_full{c}"] == res[f"tok_tp{c}"], res
        assert res["tie_full"] == 3 and res["tie_tp"] == 3, res

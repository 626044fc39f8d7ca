"""ORACLE / TEST INFRASTRUCTURE ONLY — fp32 numpy forward of the decoder the
device executes (standard Llama/Qwen math: RMSNorm, RoPE rotate-half, GQA
causal softmax attention, SwiGLU MLP, untied lm_head).

The reference has no token generation at all, so token and
logit parity is "parity unpinned" against the reference: this module is the
builder's independent restatement of the textbook math, fed the exact bf16
weights the device holds (downloaded through the C-ABI) and run in fp32.
"""
from __future__ import annotations

import numpy as np


class LlamaFP32:
    def __init__(self, dev=None, *, arch=None, weights=None):
        """From a device (weights downloaded through the C-ABI) or from an
        arch + a dict of fp32 arrays shaped like the attributes below."""
        if dev is None:
            self._init_arrays(arch, weights)
            return
        from paper_2507_06608_b200 import device as D
        a = dev.arch
        self.a = a
        self.hd = a.head_dim
        self.H, self.Hkv = a.n_heads, a.n_kv_heads
        d, f = a.hidden, a.ffn
        qkv_rows = (self.H + 2 * self.Hkv) * self.hd
        self.emb = dev.weight(D.W_EMBED).reshape(a.vocab, d)
        self.layers = []
        for l in range(a.n_layers):
            gu = dev.weight(D.W_GATE_UP, l).reshape(f // 64, 2, 64, d)
            self.layers.append(dict(
                attn_norm=dev.weight(D.W_ATTN_NORM, l),
                qkv=dev.weight(D.W_QKV, l).reshape(qkv_rows, d),
                bias=dev.weight(D.W_QKV_BIAS, l) if a.qkv_bias else None,
                o=dev.weight(D.W_O, l).reshape(d, self.H * self.hd),
                ffn_norm=dev.weight(D.W_FFN_NORM, l),
                gate=gu[:, 0].reshape(f, d), up=gu[:, 1].reshape(f, d),
                down=dev.weight(D.W_DOWN, l).reshape(d, f)))
        self.final_norm = dev.weight(D.W_FINAL_NORM)
        self.lm = dev.weight(D.W_LM_HEAD).reshape(a.vocab, d)
        self._rope_init()

    def _init_arrays(self, a, w):
        self.a = a
        self.hd = a.head_dim
        self.H, self.Hkv = w.get("H", a.n_heads), w.get("Hkv", a.n_kv_heads)
        self.emb, self.layers = w["emb"], w["layers"]
        self.final_norm, self.lm = w["final_norm"], w["lm"]
        self._rope_init()

    def _rope_init(self):
        j = np.arange(self.hd // 2, dtype=np.float64)
        self.inv_freq = (float(self.a.rope_theta) ** (-2.0 * j / self.hd)).astype(np.float32)

    def shard(self, plan) -> "LlamaFP32":
        """Megatron shard described by an nx_tp_shard (nx_tp_shard_plan):
        QKV / gate / up by output rows, O / down by input columns, lm_head by
        vocab rows [vocab0, vocab0 + vocab_valid)."""
        hd, H, Hkv = self.hd, self.a.n_heads, self.a.n_kv_heads
        q0, nq, k0, nk = plan.q_head0, plan.n_q_heads, plan.kv_head0, plan.n_kv_heads
        f0, nf = plan.ffn0, plan.ffn_local
        rows = np.concatenate([np.arange(q0 * hd, (q0 + nq) * hd),
                               H * hd + np.arange(k0 * hd, (k0 + nk) * hd),
                               (H + Hkv) * hd + np.arange(k0 * hd, (k0 + nk) * hd)])
        layers = [dict(attn_norm=L["attn_norm"], qkv=L["qkv"][rows],
                       bias=None if L["bias"] is None else L["bias"][rows],
                       o=L["o"][:, q0 * hd:(q0 + nq) * hd], ffn_norm=L["ffn_norm"],
                       gate=L["gate"][f0:f0 + nf], up=L["up"][f0:f0 + nf], down=L["down"][:, f0:f0 + nf])
                  for L in self.layers]
        sh = LlamaFP32(arch=self.a, weights=dict(
            H=nq, Hkv=nk, emb=self.emb, layers=layers, final_norm=self.final_norm,
            lm=self.lm[plan.vocab0:plan.vocab0 + plan.vocab_valid]))
        sh.rank, sh.vocab0 = plan.rank, plan.vocab0
        return sh

    def tp_greedy(self, tokens, all_reduce, all_gather):
        """One TP rank's greedy next token for the last position: the O / down
        partials are summed with all_reduce (rank 0 folds the residual in),
        each rank's (max, global argmax) pair is all-gathered and folded with
        the lowest-global-index tie rule. Test infrastructure for the
        device's NCCL / peer-memory TP path (tp.cuh)."""
        h = self.hidden(tokens, all_reduce=all_reduce, rank=self.rank)[-1:]
        lg = (h @ self.lm.T)[0]
        j = int(np.argmax(lg))
        pairs = all_gather(np.array([lg[j], self.vocab0 + j], dtype=np.float64))
        best = min(pairs, key=lambda p: (-p[0], p[1]))
        return int(best[1])

    def _norm(self, x, w):
        return x / np.sqrt((x * x).mean(-1, keepdims=True) + np.float32(self.a.rms_eps)) * w

    def _rope(self, x, pos):  # x [n, heads, hd]
        ang = pos.astype(np.float32)[:, None] * self.inv_freq[None, :]
        c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
        h = self.hd // 2
        a, b = x[..., :h], x[..., h:]
        return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)

    def logits(self, tokens: np.ndarray) -> np.ndarray:
        """Causal forward over a whole sequence; logits at every position [n, vocab]."""
        return self.hidden(tokens) @ self.lm.T

    @staticmethod
    def _residual(x, part, all_reduce, rank):
        if all_reduce is None:
            return x + part
        return all_reduce(x + part if rank == 0 else part)

    def hidden(self, tokens, all_reduce=None, rank=0) -> np.ndarray:
        """Final-normed hidden states [n, d]; all_reduce != None: TP rank."""
        tokens = np.asarray(tokens)
        n = len(tokens)
        pos = np.arange(n)
        x = self.emb[tokens].astype(np.float32)
        G = self.H // self.Hkv
        mask = np.triu(np.full((n, n), -np.inf, dtype=np.float32), 1)
        for L in self.layers:
            h = self._norm(x, L["attn_norm"])
            qkv = h @ L["qkv"].T
            if L["bias"] is not None:
                qkv = qkv + L["bias"]
            q = qkv[:, : self.H * self.hd].reshape(n, self.H, self.hd)
            k = qkv[:, self.H * self.hd: (self.H + self.Hkv) * self.hd].reshape(n, self.Hkv, self.hd)
            v = qkv[:, (self.H + self.Hkv) * self.hd:].reshape(n, self.Hkv, self.hd)
            q, k = self._rope(q, pos), self._rope(k, pos)
            out = np.empty((n, self.H, self.hd), dtype=np.float32)
            for hh in range(self.H):
                kv = hh // G
                s = (q[:, hh] @ k[:, kv].T) / np.float32(np.sqrt(self.hd)) + mask
                s = s - s.max(-1, keepdims=True)
                p = np.exp(s)
                p /= p.sum(-1, keepdims=True)
                out[:, hh] = p @ v[:, kv]
            x = self._residual(x, out.reshape(n, -1) @ L["o"].T, all_reduce, rank)
            h = self._norm(x, L["ffn_norm"])
            g, u = h @ L["gate"].T, h @ L["up"].T
            x = self._residual(x, ((g / (1 + np.exp(-g))) * u) @ L["down"].T, all_reduce, rank)
        return self._norm(x, self.final_norm)

    def greedy(self, prompt, n_new):
        toks = list(prompt)
        for _ in range(n_new):
            toks.append(int(np.argmax(self.logits(np.array(toks))[-1])))
        return toks[len(prompt):]

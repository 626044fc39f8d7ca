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
    def __init__(self, dev):
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
        j = np.arange(self.hd // 2, dtype=np.float64)
        self.inv_freq = (float(a.rope_theta) ** (-2.0 * j / self.hd)).astype(np.float32)

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
            x = x + out.reshape(n, -1) @ L["o"].T
            h = self._norm(x, L["ffn_norm"])
            g, u = h @ L["gate"].T, h @ L["up"].T
            x = x + ((g / (1 + np.exp(-g))) * u) @ L["down"].T
        return self._norm(x, self.final_norm) @ self.lm.T

    def greedy(self, prompt, n_new):
        toks = list(prompt)
        for _ in range(n_new):
            toks.append(int(np.argmax(self.logits(np.array(toks))[-1])))
        return toks[len(prompt):]

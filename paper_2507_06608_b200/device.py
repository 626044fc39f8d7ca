"""Device executor bindings: model geometry presets, the nx_device handle,
raw device buffers and the single-op GEMM entry point (C-ABI, no torch)."""
from __future__ import annotations

import ctypes as C
import importlib.util
import os
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._dev_abi import (NX_TP_NCCL, NX_TP_PEER, NX_TP_PEER_COLOCATED, Arch, BatchDesc, DeviceConfig,  # noqa: F401
                       DeviceInfo, KernelStats, TpShard)

W_EMBED, W_ATTN_NORM, W_QKV, W_QKV_BIAS, W_O, W_FFN_NORM, W_GATE_UP, W_DOWN, W_FINAL_NORM, W_LM_HEAD = range(10)


def lib():
    return _abi.lib()


def _check(rc):
    if rc != 0:
        msg = (lib().nx_last_error() or b"").decode()
        if rc == _abi.NX_ENODEV:
            raise RuntimeError(f"no usable sm_100 device: {msg}")
        raise RuntimeError(f"nexus_b200 device error {rc}: {msg}")


# ---- bf16 helpers (numpy has no bf16) ------------------------------------

def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ---- geometry presets (kernel view; head_dim fixed at 128) ----------------

def arch(hidden, n_layers, n_heads, n_kv_heads, ffn, vocab, qkv_bias=0, rope_theta=500000.0,
         rms_eps=1e-5) -> Arch:
    return Arch(hidden, n_layers, n_heads, n_kv_heads, 128, ffn, vocab, qkv_bias, rope_theta, rms_eps)


ARCH_PRESETS = {
    # C1: the reference's derive(256, 1024, 2, 4, 2) has d = 256; the kernels
    # are specialized to head_dim 128, so the kernel view is 2 heads x 128
    # (MHA, so KV bytes/token = 2*L*d*2 = 2048, identical to the cost model).
    "tiny": dict(hidden=256, n_layers=2, n_heads=2, n_kv_heads=2, ffn=1024, vocab=1024, rope_theta=10000.0),
    "llama3-8b": dict(hidden=4096, n_layers=32, n_heads=32, n_kv_heads=8, ffn=14336, vocab=128256),
    "qwen2.5-14b": dict(hidden=5120, n_layers=48, n_heads=40, n_kv_heads=8, ffn=13824, vocab=152064,
                        qkv_bias=1, rope_theta=1000000.0, rms_eps=1e-6),
    "llama3-70b": dict(hidden=8192, n_layers=80, n_heads=64, n_kv_heads=8, ffn=28672, vocab=128256),
}


def arch_preset(name: str, **over) -> Arch:
    kw = dict(ARCH_PRESETS[name])
    kw.update(over)
    return arch(**kw)


def _prefer_torch_nccl():
    """Point NX_NCCL_LIB at the libnccl torch links (the pip nvidia-nccl
    wheel) so both share one NCCL; loading the system copy first under the
    same soname would break a later `import torch`."""
    if os.environ.get("NX_NCCL_LIB"):
        return
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        so = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(so):
            os.environ["NX_NCCL_LIB"] = so
            return


_prefer_torch_nccl()

# Each lane of each rank is its own stream; with the default 8 hardware
# work queues, 16+ streams (TP=8 colocated: 8 ranks x 2 lanes) alias queues,
# and a rank's spinning peer all-reduce can then sit in front of the very
# kernel it waits for. Read by the driver at context creation (C++ hosts that
# drive colocated TP groups set it themselves).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def shard_plan(a: Arch, tp_size: int, rank: int) -> TpShard:
    """nx_tp_shard_plan: the heads / ffn features / vocab rows rank owns."""
    s = TpShard()
    _check(lib().nx_tp_shard_plan(C.byref(a), tp_size, rank, C.byref(s)))
    return s


def tp_follow(dev, recv) -> int:
    """Follower loop of an NX_TP_NCCL group served on rank 0's device clock.

    Rank 0's engine forwards every launch (Engine.set_launch_observer) and
    this loop replays it on the follower's shard: `recv()` returns the next
    batch (the batch_from_desc dict) or None at the end. A lane's next batch
    is launched after that lane's previous one finished, exactly as on rank
    0, so every rank issues the same batches in the same per-lane order and
    the per-lane NCCL collectives pair up. Returns the number of launches."""
    pending, n = set(), 0
    while True:
        b = recv()
        if b is None:
            break
        lane = b["lane"]
        if lane in pending:
            dev.wait(lane)
        dev.launch(b["members"], lane=lane, sm_pct=b["sm_pct"])
        pending.add(lane)
        n += 1
    for lane in sorted(pending):
        dev.wait(lane)
    return n


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().nx_nccl_unique_id(buf))
    return bytes(buf)


class Device:
    """nx_device: weights + paged KV cache + per-lane workspaces + SM layouts."""

    def __init__(self, a: Arch, *, num_pages=4096, page_tokens=16, max_prefill_tokens=2048 + 64,
                 max_decode_batch=64, green_contexts=True, seed=1, weight_gain=1.0, lm_head_gain=4.0,
                 device=0, tp_size=1, tp_rank=0, tp_mode=NX_TP_NCCL, nccl_ids=None):
        """tp_size > 1, tp_mode NX_TP_NCCL: this process holds shard ``tp_rank``
        of a Megatron-style tensor-parallel model; ``nccl_ids`` are the two
        128-byte ids from ``nccl_unique_id()`` on rank 0 (one communicator per
        lane), shared by the caller (e.g. torch.distributed.broadcast_object_list).
        tp_mode NX_TP_PEER / NX_TP_PEER_COLOCATED: this Device drives all
        ranks (GPUs device..device+tp-1, or all on ``device``) with
        peer-memory collectives."""
        self.arch = a
        cfg = DeviceConfig(a, device, page_tokens, num_pages, max_prefill_tokens, max_decode_batch,
                           1 if green_contexts else 0, seed, weight_gain, lm_head_gain, tp_size, tp_rank,
                           tp_mode)
        if tp_size > 1 and tp_mode == NX_TP_NCCL:
            if nccl_ids is None or len(nccl_ids) != 2:
                raise ValueError("tp_size > 1 needs two NCCL unique ids")
            for lane in range(2):
                C.memmove(C.addressof(cfg.nccl_id[lane]), bytes(nccl_ids[lane]), 128)
        self.tp = shard_plan(a, tp_size, tp_rank)
        self.cfg = cfg
        self.handle = C.c_void_p()
        _check(lib().nx_device_create(C.byref(cfg), C.byref(self.handle)))

    def info(self) -> DeviceInfo:
        i = DeviceInfo()
        _check(lib().nx_device_get_info(self.handle, C.byref(i)))
        return i

    def set_profiling(self, sample_every: int) -> None:
        _check(lib().nx_device_set_profiling(self.handle, sample_every))

    def kernel_stats(self) -> KernelStats:
        k = KernelStats()
        _check(lib().nx_device_kernel_stats(self.handle, C.byref(k)))
        return k

    def reset_kernel_stats(self) -> None:
        _check(lib().nx_device_reset_kernel_stats(self.handle))

    def weight(self, tensor: int, layer: int = 0) -> np.ndarray:
        n = C.c_size_t()
        _check(lib().nx_device_weight(self.handle, tensor, layer, None, 0, C.byref(n)))
        out = np.empty(n.value // 2, dtype=np.uint16)
        if n.value:
            _check(lib().nx_device_weight(self.handle, tensor, layer, out.ctypes.data, n.value, C.byref(n)))
        return bf16_to_f32(out)

    def _desc(self, members, lane, sm_pct):
        n = len(members)
        nt = (C.c_int32 * n)(*[len(m["tokens"]) for m in members])
        sp = (C.c_int64 * n)(*[m["start"] for m in members])
        sa = (C.c_int32 * n)(*[1 if m.get("sample", True) else 0 for m in members])
        toks = [t for m in members for t in m["tokens"]]
        tk = (C.c_int32 * max(1, len(toks)))(*toks)
        npg = (C.c_int32 * n)(*[len(m["pages"]) for m in members])
        pgs = [p for m in members for p in m["pages"]]
        pg = (C.c_int32 * max(1, len(pgs)))(*pgs)
        keep = (nt, sp, sa, tk, npg, pg)
        return BatchDesc(lane, sm_pct, n, 0, nt, sp, sa, tk, npg, pg), keep, int(sum(sa))

    def launch(self, members, lane=0, sm_pct=100):
        """Asynchronous launch (returns immediately); pair with wait(lane)."""
        b, keep, ns = self._desc(members, lane, sm_pct)
        _check(lib().nx_device_launch(self.handle, C.byref(b)))
        self._pending = getattr(self, "_pending", {})
        self._pending[lane] = ns

    def wait(self, lane):
        ns = self._pending.pop(lane)
        out = (C.c_int32 * max(1, ns))()
        ms = C.c_double()
        _check(lib().nx_device_wait(self.handle, lane, out, None, C.byref(ms)))
        return list(out[:ns]), ms.value

    def forward(self, members, lane=0, sm_pct=100, want_logits=False):
        """members: list of dict(tokens=[...], start=int, pages=[...], sample=bool)."""
        n = len(members)
        nt = (C.c_int32 * n)(*[len(m["tokens"]) for m in members])
        sp = (C.c_int64 * n)(*[m["start"] for m in members])
        sa = (C.c_int32 * n)(*[1 if m.get("sample", True) else 0 for m in members])
        toks = [t for m in members for t in m["tokens"]]
        tk = (C.c_int32 * max(1, len(toks)))(*toks)
        npg = (C.c_int32 * n)(*[len(m["pages"]) for m in members])
        pgs = [p for m in members for p in m["pages"]]
        pg = (C.c_int32 * max(1, len(pgs)))(*pgs)
        b = BatchDesc(lane, sm_pct, n, 0, nt, sp, sa, tk, npg, pg)
        ns = sum(sa)
        out = (C.c_int32 * max(1, ns))()
        local = self.tp.tp_size > 1 and self.cfg.tp_mode == NX_TP_NCCL
        logits = np.zeros((max(1, ns), self.tp.vocab_local if local else self.arch.vocab),
                          dtype=np.float32) if want_logits else None
        ms = C.c_double()
        _check(lib().nx_device_forward(self.handle, C.byref(b), out,
                                       logits.ctypes.data_as(C.POINTER(C.c_float)) if want_logits else None,
                                       C.byref(ms)))
        toks_out = list(out[:ns])
        return (toks_out, logits[:ns] if want_logits else None, ms.value)

    def close(self):
        if getattr(self, "handle", None):
            lib().nx_device_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()


# ---- raw buffers + single-op entry points --------------------------------

class Buf:
    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        self.nbytes = nbytes
        _check(lib().nx_dev_malloc(max(nbytes, 16), C.byref(self.ptr)))

    @classmethod
    def from_array(cls, a: np.ndarray) -> "Buf":
        a = np.ascontiguousarray(a)
        b = cls(a.nbytes)
        _check(lib().nx_dev_h2d(b.ptr, a.ctypes.data, a.nbytes))
        return b

    def to_array(self, shape, dtype) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        _check(lib().nx_dev_d2h(out.ctypes.data, self.ptr, out.nbytes))
        return out

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().nx_dev_free(self.ptr)
            self.ptr = None


EPI_STORE, EPI_BIAS, EPI_RESIDUAL, EPI_BIAS_RESIDUAL, EPI_SWIGLU, EPI_F32 = 0, 1, 2, 3, 4, 6
EPI_DECODE_FOLD = 16  # decode GEMM (tokens <= 128): stream-K fold planes -> fp32 out
EPI_DECODE_F32 = 17   # decode GEMM, direct fp32 out (data-parallel)


def gemm(x: Buf, w: Buf, tokens: int, rows: int, K: int, mode: int, out: Buf, ldo: int,
         bias: Buf | None = None, residual: Buf | None = None, ldr: int = 0, sm_count: int = 0,
         splits: int = 0, iters: int = 1) -> float:
    ms = C.c_float()
    _check(lib().nx_op_gemm(x.ptr, w.ptr, tokens, rows, K, mode, out.ptr, ldo,
                            bias.ptr if bias else None, residual.ptr if residual else None, ldr,
                            sm_count, splits, iters, C.byref(ms)))
    return ms.value

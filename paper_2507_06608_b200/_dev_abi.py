"""ctypes prototypes for the device half of include/nexus_b200.h."""
from __future__ import annotations

import ctypes as C

P = C.POINTER
sz = C.c_size_t


class Arch(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("qkv_bias", C.c_int32), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float)]


class DeviceConfig(C.Structure):
    _fields_ = [("arch", Arch), ("device", C.c_int32), ("page_tokens", C.c_int32),
                ("num_pages", C.c_int32), ("max_prefill_tokens", C.c_int32),
                ("max_decode_batch", C.c_int32), ("green_contexts", C.c_int32),
                ("weight_seed", C.c_uint64), ("weight_gain", C.c_float), ("lm_head_gain", C.c_float),
                ("tp_size", C.c_int32), ("tp_rank", C.c_int32), ("tp_mode", C.c_int32), ("tp_pad", C.c_int32),
                ("nccl_id", (C.c_uint8 * 128) * 2)]


NX_TP_NCCL, NX_TP_PEER, NX_TP_PEER_COLOCATED = 0, 1, 2


class TpShard(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("tp_size", "rank", "q_head0", "n_q_heads", "kv_head0", "n_kv_heads",
                                         "ffn0", "ffn_local", "vocab0", "vocab_local", "vocab_valid",
                                         "vocab_padded")]


class DeviceInfo(C.Structure):
    _fields_ = [("sm_count", C.c_int32), ("n_layouts", C.c_int32),
                ("layout_decode_sms", C.c_int32 * 32), ("layout_prefill_sms", C.c_int32 * 32),
                ("weight_bytes", C.c_uint64), ("kv_bytes", C.c_uint64), ("workspace_bytes", C.c_uint64)]


class BatchDesc(C.Structure):
    _fields_ = [("lane", C.c_int32), ("sm_pct", C.c_int32), ("n_members", C.c_int32), ("_pad0", C.c_int32),
                ("n_tokens", P(C.c_int32)), ("start_pos", P(C.c_int64)), ("sample", P(C.c_int32)),
                ("tokens", P(C.c_int32)), ("n_pages", P(C.c_int32)), ("pages", P(C.c_int32))]


class KernelStats(C.Structure):
    _fields_ = [("ms", C.c_double * 5), ("bytes", C.c_double * 5), ("flops", C.c_double * 5),
                ("launches", C.c_uint64 * 5), ("batches_sampled", C.c_uint64),
                ("batch_ms_sampled", C.c_double), ("kernel_launches", C.c_uint64),
                ("batches", C.c_uint64), ("sm_ms", C.c_double * 5), ("op_ms", C.c_double * 5),
                ("op_launches", C.c_uint64 * 5)]


PROTOS = {
    "nx_tp_shard_plan": (C.c_int, [P(Arch), C.c_int32, C.c_int32, P(TpShard)]),
    "nx_nccl_unique_id": (C.c_int, [P(C.c_uint8)]),
    "nx_device_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
    "nx_device_kernel_stats": (C.c_int, [C.c_void_p, P(KernelStats)]),
    "nx_device_reset_kernel_stats": (C.c_int, [C.c_void_p]),
    "nx_device_create": (C.c_int, [P(DeviceConfig), P(C.c_void_p)]),
    "nx_device_destroy": (None, [C.c_void_p]),
    "nx_device_get_info": (C.c_int, [C.c_void_p, P(DeviceInfo)]),
    "nx_engine_bind_device": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nx_device_weight": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, sz, P(sz)]),
    "nx_device_forward": (C.c_int, [C.c_void_p, P(BatchDesc), P(C.c_int32), P(C.c_float), P(C.c_double)]),
    "nx_device_launch": (C.c_int, [C.c_void_p, P(BatchDesc)]),
    "nx_device_wait": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_int32), P(C.c_float), P(C.c_double)]),
    "nx_dev_malloc": (C.c_int, [sz, P(C.c_void_p)]),
    "nx_dev_free": (C.c_int, [C.c_void_p]),
    "nx_dev_h2d": (C.c_int, [C.c_void_p, C.c_void_p, sz]),
    "nx_dev_d2h": (C.c_int, [C.c_void_p, C.c_void_p, sz]),
    "nx_dev_sync": (C.c_int, []),
    "nx_op_gemm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                             C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                             P(C.c_float)]),
}


def bind_all(lib: C.CDLL) -> None:
    for name, (res, args) in PROTOS.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.restype, fn.argtypes = res, args

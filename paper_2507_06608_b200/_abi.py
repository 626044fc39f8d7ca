"""ctypes mirror of include/nexus_b200.h (POD structs + prototypes).

Used by the package API (``paper_2507_06608_b200``) to call the product
library ``libnexus_b200.so`` and by the test oracle to call the reference
shim ``oracle/_ref/libnexussim_ref.so`` with the same structs.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB_PATH = os.environ.get("NX_LIB_PATH") or os.path.join(HERE, "libnexus_b200.so")  # override: A/B experiments

NX_OK, NX_EINVAL, NX_ERUNTIME, NX_ENOMEM, NX_EAGAIN, NX_EDONE, NX_ENODEV = range(7)
NX_ENGINE_NEXUS, NX_ENGINE_MONOLITHIC, NX_ENGINE_STATIC = 0, 1, 2
NX_PREFILL_SPF, NX_PREFILL_FCFS = 0, 1
NX_CLOCK_VIRTUAL, NX_CLOCK_DEVICE, NX_CLOCK_REPLAY = 0, 1, 2
NX_OP_QKV_PROJ, NX_OP_ATTN_PREFILL, NX_OP_ATTN_DECODE, NX_OP_ATTN_OUT_PROJ, NX_OP_FFN = range(5)
NX_MODE_PREFILL, NX_MODE_DECODE = 0, 1
NX_PHASE_PREFILL, NX_PHASE_DECODE = 0, 1
NX_MAX_OPS = 8


class ModelConfig(C.Structure):
    _fields_ = [("hidden_dim", C.c_int64), ("ffn_dim", C.c_int64), ("num_layers", C.c_int32),
                ("num_heads", C.c_int32), ("element_bytes", C.c_int32), ("_pad0", C.c_int32),
                ("kv_bytes_per_token", C.c_int64), ("weight_bytes_per_layer_dense", C.c_int64),
                ("weight_bytes_per_layer_attn", C.c_int64)]


class GpuSpec(C.Structure):
    _fields_ = [("total_sm", C.c_int32), ("_pad0", C.c_int32), ("peak_compute", C.c_double),
                ("peak_bandwidth", C.c_double), ("kv_capacity_bytes", C.c_int64)]


class SaturationCurve(C.Structure):
    _fields_ = [("r_sat", C.c_double), ("lambda_", C.c_double)]


class KernelProfile(C.Structure):
    _fields_ = [("qkv_proj", SaturationCurve), ("attn_prefill", SaturationCurve),
                ("attn_decode", SaturationCurve), ("attn_out_proj", SaturationCurve),
                ("ffn", SaturationCurve)]


class ControllerConfig(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("kv_switch_fraction", C.c_double),
                ("gamma", C.c_double), ("delta_pp", C.c_int32), ("max_decode_batch", C.c_int32),
                ("chunk_size", C.c_int64), ("token_budget", C.c_int64)]


class PartitionState(C.Structure):
    _fields_ = [("r_p", C.c_int32), ("r_d", C.c_int32), ("last_applied_r_p", C.c_int32)]


class EngineConfig(C.Structure):
    _fields_ = [("kind", C.c_int32), ("static_r_p", C.c_int32), ("prefill_policy", C.c_int32),
                ("clock_mode", C.c_int32), ("timeout_sim_s", C.c_double),
                ("max_events", C.c_uint64)]


class CostExt(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("contention", C.c_int32), ("bw_sat", C.c_double * 5),
                ("contention_c", C.c_double * 3), ("decode_target_s", C.c_double)]


class SimConfig(C.Structure):
    _fields_ = [("model", ModelConfig), ("gpu", GpuSpec), ("ctrl", ControllerConfig),
                ("profile", KernelProfile), ("engine", EngineConfig), ("ext", CostExt)]


class Request(C.Structure):
    _fields_ = [("id", C.c_uint64), ("arrival_s", C.c_double), ("prompt_len", C.c_int64),
                ("output_len", C.c_int64)]


class OpWorkload(C.Structure):
    _fields_ = [("kind", C.c_int32), ("is_attention", C.c_int32), ("flops", C.c_double),
                ("mem_bytes", C.c_double), ("kv_bytes", C.c_double)]


class OpLatency(C.Structure):
    _fields_ = [("kind", C.c_int32), ("memory_bound", C.c_int32), ("compute_s", C.c_double),
                ("mem_s", C.c_double)]


class Breakdown(C.Structure):
    _fields_ = [("total_s", C.c_double), ("attn_mem_time_s", C.c_double), ("n_ops", C.c_int32),
                ("_pad0", C.c_int32), ("per_op", OpLatency * NX_MAX_OPS)]


LATENCY_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_int32)


class PhaseModel(C.Structure):
    _fields_ = [("active", C.c_int32), ("latency_at", LATENCY_FN), ("user", C.c_void_p)]


class AdjustOutcome(C.Structure):
    _fields_ = [("r_p", C.c_int32), ("r_d", C.c_int32), ("infeasible", C.c_int32),
                ("queries", C.c_int32)]


class Decision(C.Structure):
    _fields_ = [("r_p", C.c_int32), ("r_d", C.c_int32), ("mode", C.c_int32),
                ("switched", C.c_int32), ("infeasible", C.c_int32), ("candidate_r_p", C.c_int32),
                ("iterations_searched", C.c_int32), ("_pad0", C.c_int32)]


class PrefillEntry(C.Structure):
    _fields_ = [("id", C.c_uint64), ("remaining", C.c_int64), ("arrival_s", C.c_double)]


class DecodeCandidate(C.Structure):
    _fields_ = [("id", C.c_uint64), ("arrival_s", C.c_double)]


class BatchMember(C.Structure):
    _fields_ = [("id", C.c_uint64), ("tokens", C.c_int64)]


class EngineStats(C.Structure):
    _fields_ = [("events", C.c_uint64), ("decisions", C.c_uint64), ("switches", C.c_uint64),
                ("launches", C.c_uint64), ("completed_requests", C.c_uint64),
                ("timed_out", C.c_int32), ("current_r_p", C.c_int32), ("clock_s", C.c_double),
                ("kv_used", C.c_int64), ("kv_reserved", C.c_int64), ("kv_capacity", C.c_int64)]


class RequestState(C.Structure):
    _fields_ = [("id", C.c_uint64), ("arrival_s", C.c_double), ("prompt_len", C.c_int64),
                ("output_len", C.c_int64), ("prefilled_len", C.c_int64),
                ("decoded_len", C.c_int64), ("first_token_s", C.c_double),
                ("finish_s", C.c_double)]


class Goodput(C.Structure):
    _fields_ = [("completed", C.c_uint64), ("slo_met", C.c_uint64), ("makespan_s", C.c_double),
                ("goodput_tok_s", C.c_double), ("output_tokens", C.c_double),
                ("ttft_p50", C.c_double), ("ttft_p99", C.c_double), ("tbt_p50", C.c_double),
                ("tbt_p99", C.c_double)]


P = C.POINTER
sz = C.c_size_t
_PROTOS = {
    # name: (restype, argtypes)
    "nx_last_error": (C.c_char_p, []),
    "nx_version": (C.c_char_p, []),
    "nx_sim_config_size": (C.c_size_t, []),
    "nx_model_derive": (ModelConfig, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32]),
    "nx_controller_config_default": (ControllerConfig, []),
    "nx_kernel_profile_default": (KernelProfile, []),
    "nx_engine_config_default": (EngineConfig, []),
    "nx_validate_config": (C.c_int, [P(ModelConfig), P(GpuSpec), P(ControllerConfig),
                                     P(KernelProfile), C.c_char_p, sz]),
    "nx_prefill_batch_workloads": (C.c_int, [P(ModelConfig), P(C.c_int64), P(C.c_int64), sz,
                                             P(OpWorkload), P(sz)]),
    "nx_decode_op_workloads": (C.c_int, [P(ModelConfig), P(C.c_int64), sz, P(OpWorkload), P(sz)]),
    "nx_mixed_batch_workloads": (C.c_int, [P(ModelConfig), P(C.c_int64), P(C.c_int64), sz,
                                           P(C.c_int64), sz, P(OpWorkload), P(sz)]),
    "nx_compute_latency": (C.c_int, [C.c_double, C.c_double, SaturationCurve, C.c_double,
                                     P(C.c_double)]),
    "nx_phase_latency_isolated": (C.c_int, [P(OpWorkload), sz, C.c_double, P(GpuSpec),
                                            P(KernelProfile), P(Breakdown)]),
    "nx_effective_decode_bandwidth": (C.c_int, [C.c_double] * 5 + [P(C.c_double)]),
    "nx_decode_latency_contended": (C.c_int, [P(OpWorkload), sz, C.c_double, P(Breakdown),
                                              P(OpWorkload), sz, P(GpuSpec), P(KernelProfile),
                                              P(Breakdown)]),
    "nx_set_cost_ext": (C.c_int, [C.c_void_p]),
    "nx_min_phase_latency": (C.c_double, [P(OpWorkload), sz, P(GpuSpec), P(KernelProfile)]),
    "nx_select_mode": (C.c_int, [C.c_int64, C.c_int64, C.c_double]),
    "nx_adjust_partition": (C.c_int, [C.c_int32, P(PartitionState), P(PhaseModel),
                                      P(PhaseModel), P(ControllerConfig), P(AdjustOutcome)]),
    "nx_controller_create": (C.c_int, [P(PartitionState), P(ControllerConfig), P(C.c_void_p)]),
    "nx_controller_destroy": (None, [C.c_void_p]),
    "nx_controller_decide": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(PhaseModel),
                                       P(PhaseModel), P(Decision)]),
    "nx_controller_state": (C.c_int, [C.c_void_p, P(PartitionState)]),
    "nx_spf_schedule": (C.c_int, [P(PrefillEntry), sz, C.c_int64, C.c_double, C.c_double,
                                  C.c_int32, P(BatchMember), sz, P(sz), P(C.c_int64)]),
    "nx_fcfs_prefill_schedule": (C.c_int, [P(PrefillEntry), sz, C.c_int64, P(BatchMember), sz,
                                           P(sz), P(C.c_int64)]),
    "nx_fcfs_decode_schedule": (C.c_int, [P(DecodeCandidate), sz, C.c_int32, P(BatchMember), sz,
                                          P(sz), P(C.c_int64)]),
    "nx_chunked_mixed_schedule": (C.c_int, [P(PrefillEntry), sz, P(DecodeCandidate), sz,
                                            C.c_int64, C.c_int32, C.c_int64, P(BatchMember), sz,
                                            P(sz), P(C.c_int64)]),
    "nx_workload_preset_trace": (C.c_int, [C.c_char_p, C.c_double, C.c_int64, C.c_uint64,
                                           P(Request), sz, P(sz)]),
    "nx_trace_to_text": (C.c_int, [P(Request), sz, C.c_char_p, sz, P(sz)]),
    "nx_trace_from_text": (C.c_int, [C.c_char_p, P(Request), sz, P(sz)]),
    "nx_kernel_profile_to_text": (C.c_int, [P(KernelProfile), C.c_char_p, sz, P(sz)]),
    "nx_kernel_profile_from_text": (C.c_int, [C.c_char_p, P(KernelProfile), C.c_char_p, sz]),
    "nx_engine_create": (C.c_int, [P(SimConfig), P(C.c_void_p)]),
    "nx_engine_destroy": (None, [C.c_void_p]),
    "nx_engine_last_error": (C.c_char_p, [C.c_void_p]),
    "nx_submit": (C.c_int, [C.c_void_p, P(Request)]),
    "nx_submit_trace": (C.c_int, [C.c_void_p, P(Request), sz]),
    "nx_submit_with_tokens": (C.c_int, [C.c_void_p, P(Request), P(C.c_int32)]),
    "nx_step": (C.c_int, [C.c_void_p]),
    "nx_run": (C.c_int, [C.c_void_p]),
    "nx_engine_set_replay_latencies": (C.c_int, [C.c_void_p, P(C.c_double), sz]),
    "nx_engine_set_logging": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "nx_engine_set_slo": (C.c_int, [C.c_void_p, C.c_double, C.c_double]),
    "nx_engine_set_launch_observer": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "nx_engine_get_stats": (C.c_int, [C.c_void_p, P(EngineStats)]),
    "nx_engine_event_log": (C.c_int, [C.c_void_p, C.c_char_p, sz, P(sz)]),
    "nx_engine_decision_log": (C.c_int, [C.c_void_p, C.c_char_p, sz, P(sz)]),
    "nx_engine_summary_json": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, sz, P(sz)]),
    "nx_engine_goodput": (C.c_int, [C.c_void_p, P(Goodput)]),
    "nx_engine_launch_latencies": (C.c_int, [C.c_void_p, P(C.c_double), sz, P(sz)]),
    "nx_engine_launch_device_ms": (C.c_int, [C.c_void_p, P(C.c_double), sz, P(sz)]),
    "nx_engine_requests": (C.c_int, [C.c_void_p, P(RequestState), sz, P(sz)]),
    "nx_engine_token_times": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_double), sz, P(sz)]),
    "nx_engine_tokens": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_int32), sz, P(sz)]),
    "nx_kv_usage": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64)]),
    "nx_kv_block_table": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_int32), sz, P(sz)]),
    "nx_kv_page_log": (C.c_int, [C.c_void_p, C.c_char_p, sz, P(sz)]),
    "nx_kv_configure": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
}


def header_symbols(path: str | None = None) -> list[str]:
    """Function names declared in include/nexus_b200.h (for the export test)."""
    import re
    path = path or os.path.join(REPO, "include", "nexus_b200.h")
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(nx_[a-z0-9_]+)\s*\(", text)
    return sorted(set(n for n in names if not n.endswith("_t")))


def bind(lib: C.CDLL, protos: dict, prefix_from: str = "nx_", prefix_to: str = "nx_") -> None:
    for name, (res, args) in protos.items():
        fname = prefix_to + name[len(prefix_from):]
        fn = getattr(lib, fname, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args


_lib = None


def lib() -> C.CDLL:
    """The product library; raises (never falls back) if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `make -C paper_2507_06608_b200` "
                               "or __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        bind(_lib, _PROTOS)
        _bind_device(_lib)
    return _lib


def _bind_device(l: C.CDLL) -> None:
    try:
        from . import _dev_abi
    except ImportError:  # device prototypes are added with the CUDA library
        return
    _dev_abi.bind_all(l)

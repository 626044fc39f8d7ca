"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes binding of the unmodified reference library (nexussim core, built by
oracle/Makefile into oracle/_ref/libnexussim_ref.so). Only tests/,
__graft_entry__.smoke() and bench.py's reference / cpu_baseline legs import
this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF_SO = os.path.join(HERE, "_ref", "libnexussim_ref.so")
REF_SRC = "/root/reference/proj/core"

sys.path.insert(0, REPO)
from paper_2507_06608_b200 import _abi  # noqa: E402  (shared POD struct definitions)
from paper_2507_06608_b200._abi import (BatchMember, Breakdown, DecodeCandidate,  # noqa: E402
                                        OpWorkload, PrefillEntry, Request)

_lib = None


def build() -> bool:
    """Compile the reference (only possible where /root/reference exists)."""
    if not os.path.isdir(REF_SRC):
        return os.path.exists(REF_SO)
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)
    return True


def available() -> bool:
    return os.path.exists(REF_SO)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(REF_SO):
            build()
        _lib = C.CDLL(REF_SO)
        P, sz = C.POINTER, C.c_size_t
        protos = {
            "nxref_last_error": (C.c_char_p, []),
            "nxref_free": (None, [C.c_void_p]),
            "nxref_model_derive": (_abi.ModelConfig, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32]),
            "nxref_defaults": (None, [P(_abi.ControllerConfig), P(_abi.KernelProfile), P(_abi.EngineConfig)]),
            "nxref_model_preset": (C.c_int, [C.c_char_p, P(_abi.ModelConfig)]),
            "nxref_gpu_preset": (C.c_int, [C.c_char_p, P(_abi.GpuSpec)]),
            "nxref_validate_config": (C.c_int, [P(_abi.ModelConfig), P(_abi.GpuSpec), P(_abi.ControllerConfig),
                                                P(_abi.KernelProfile), C.c_char_p, sz]),
            "nxref_prefill_batch_workloads": (C.c_int, [P(_abi.ModelConfig), P(C.c_int64), P(C.c_int64), sz,
                                                        P(OpWorkload), P(sz)]),
            "nxref_decode_op_workloads": (C.c_int, [P(_abi.ModelConfig), P(C.c_int64), sz, P(OpWorkload), P(sz)]),
            "nxref_mixed_batch_workloads": (C.c_int, [P(_abi.ModelConfig), P(C.c_int64), P(C.c_int64), sz,
                                                      P(C.c_int64), sz, P(OpWorkload), P(sz)]),
            "nxref_compute_latency": (C.c_int, [C.c_double, C.c_double, _abi.SaturationCurve, C.c_double,
                                                P(C.c_double)]),
            "nxref_phase_latency_isolated": (C.c_int, [P(OpWorkload), sz, C.c_double, P(_abi.GpuSpec),
                                                       P(_abi.KernelProfile), P(Breakdown)]),
            "nxref_effective_decode_bandwidth": (C.c_int, [C.c_double] * 5 + [P(C.c_double)]),
            "nxref_decode_latency_contended": (C.c_int, [P(OpWorkload), sz, C.c_double, P(Breakdown),
                                                         P(OpWorkload), sz, P(_abi.GpuSpec),
                                                         P(_abi.KernelProfile), P(Breakdown)]),
            "nxref_min_phase_latency": (C.c_double, [P(OpWorkload), sz, P(_abi.GpuSpec), P(_abi.KernelProfile)]),
            "nxref_select_mode": (C.c_int, [C.c_int64, C.c_int64, C.c_double]),
            "nxref_adjust_partition": (C.c_int, [C.c_int32, P(_abi.PartitionState), P(_abi.PhaseModel),
                                                 P(_abi.PhaseModel), P(_abi.ControllerConfig),
                                                 P(_abi.AdjustOutcome)]),
            "nxref_controller_create": (C.c_int, [P(_abi.PartitionState), P(_abi.ControllerConfig),
                                                  P(C.c_void_p)]),
            "nxref_controller_destroy": (None, [C.c_void_p]),
            "nxref_controller_decide": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(_abi.PhaseModel),
                                                  P(_abi.PhaseModel), P(_abi.Decision)]),
            "nxref_spf_schedule": (C.c_int, [P(PrefillEntry), sz, C.c_int64, C.c_double, C.c_double, C.c_int32,
                                             P(BatchMember), sz, P(sz), P(C.c_int64)]),
            "nxref_fcfs_prefill_schedule": (C.c_int, [P(PrefillEntry), sz, C.c_int64, P(BatchMember), sz,
                                                      P(sz), P(C.c_int64)]),
            "nxref_fcfs_decode_schedule": (C.c_int, [P(DecodeCandidate), sz, C.c_int32, P(BatchMember), sz,
                                                     P(sz), P(C.c_int64)]),
            "nxref_chunked_mixed_schedule": (C.c_int, [P(PrefillEntry), sz, P(DecodeCandidate), sz, C.c_int64,
                                                       C.c_int32, C.c_int64, P(BatchMember), sz, P(sz),
                                                       P(C.c_int64)]),
            "nxref_workload_preset_trace": (C.c_int, [C.c_char_p, C.c_double, C.c_int64, C.c_uint64,
                                                      P(Request), sz, P(sz)]),
            "nxref_trace_text": (C.c_int, [P(Request), sz, P(C.c_void_p)]),
            "nxref_kernel_profile_text": (C.c_int, [P(_abi.KernelProfile), P(C.c_void_p)]),
            "nxref_kernel_profile_load_text": (C.c_int, [C.c_char_p, P(_abi.KernelProfile), P(C.c_void_p)]),
            "nxref_run": (C.c_int, [P(_abi.SimConfig), P(Request), sz, P(C.c_void_p), P(C.c_void_p),
                                    P(C.c_void_p), P(C.c_double), P(C.c_int32)]),
            "nxref_replay_summary": (C.c_int, [C.c_char_p, C.c_char_p, P(C.c_void_p)]),
        }
        for name, (res, args) in protos.items():
            fn = getattr(_lib, name)
            fn.restype, fn.argtypes = res, args
    return _lib


def _take(p: C.c_void_p) -> str:
    if not p.value:
        return ""
    s = C.string_at(p.value).decode()
    lib().nxref_free(p)
    return s


def _check(rc):
    if rc != 0:
        raise ValueError(lib().nxref_last_error().decode())


def run(cfg: _abi.SimConfig, trace) -> dict:
    """nexus::run over the trace; returns the logs and summary JSON text."""
    arr = (Request * max(1, len(trace)))(*trace)
    ev, dec, summ = C.c_void_p(), C.c_void_p(), C.c_void_p()
    end, to = C.c_double(), C.c_int32()
    _check(lib().nxref_run(C.byref(cfg), arr, len(trace), C.byref(ev), C.byref(dec), C.byref(summ),
                           C.byref(end), C.byref(to)))
    return {"event_log": _take(ev), "decision_log": _take(dec), "summary_json": _take(summ),
            "sim_end_s": end.value, "timed_out": bool(to.value)}


def workload_trace(preset: str, rate: float, count: int, seed: int) -> list[Request]:
    out = (Request * max(1, count))()
    n = C.c_size_t()
    _check(lib().nxref_workload_preset_trace(preset.encode(), rate, count, seed, out, count, C.byref(n)))
    return list(out[: n.value])


def trace_text(trace) -> str:
    arr = (Request * max(1, len(trace)))(*trace)
    p = C.c_void_p()
    _check(lib().nxref_trace_text(arr, len(trace), C.byref(p)))
    return _take(p)


def model_preset(name: str) -> _abi.ModelConfig:
    m = _abi.ModelConfig()
    _check(lib().nxref_model_preset(name.encode(), C.byref(m)))
    return m


def model_derive(hidden_dim: int, ffn_dim: int, num_layers: int, num_heads: int,
                 element_bytes: int = 2) -> _abi.ModelConfig:
    """ModelConfig::derive (domain.cpp:7-24) computed by the reference itself."""
    return lib().nxref_model_derive(hidden_dim, ffn_dim, num_layers, num_heads, element_bytes)


def defaults() -> tuple[_abi.ControllerConfig, _abi.KernelProfile, _abi.EngineConfig]:
    """Default-constructed ControllerConfig / KernelProfile / EngineConfig of the reference."""
    c, p, e = _abi.ControllerConfig(), _abi.KernelProfile(), _abi.EngineConfig()
    lib().nxref_defaults(C.byref(c), C.byref(p), C.byref(e))
    return c, p, e


def load_kernel_profile_text(text: str) -> tuple[_abi.KernelProfile, list[str]]:
    """load_kernel_profile (presets.cpp:128-170) through the reference loader."""
    p, w = _abi.KernelProfile(), C.c_void_p()
    rc = lib().nxref_kernel_profile_load_text(text.encode(), C.byref(p), C.byref(w))
    if rc != 0:
        raise RuntimeError(lib().nxref_last_error().decode())
    return p, [x for x in _take(w).splitlines() if x]


def kernel_profile_text(p: _abi.KernelProfile) -> str:
    """kernel_profile_text (presets.cpp:109-126) of the reference."""
    out = C.c_void_p()
    _check(lib().nxref_kernel_profile_text(C.byref(p), C.byref(out)))
    return _take(out)


def sim_config(model: _abi.ModelConfig, gpu: _abi.GpuSpec, *, kind: int = _abi.NX_ENGINE_NEXUS,
               static_r_p: int = 50, ctrl: _abi.ControllerConfig | None = None,
               profile: _abi.KernelProfile | None = None) -> _abi.SimConfig:
    """A SimConfig built from reference defaults only (no product library involved)."""
    c, p, e = defaults()
    cfg = _abi.SimConfig()
    cfg.model, cfg.gpu = model, gpu
    cfg.ctrl = ctrl if ctrl is not None else c
    cfg.profile = profile if profile is not None else p
    e.kind, e.static_r_p = kind, static_r_p
    cfg.engine = e
    return cfg


def gpu_preset(name: str) -> _abi.GpuSpec:
    g = _abi.GpuSpec()
    _check(lib().nxref_gpu_preset(name.encode(), C.byref(g)))
    return g


def replay_summary(event_log: str, label: str = "replay") -> str:
    p = C.c_void_p()
    _check(lib().nxref_replay_summary(event_log.encode(), label.encode(), C.byref(p)))
    return _take(p)

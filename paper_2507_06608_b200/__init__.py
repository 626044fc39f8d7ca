"""B200-native Nexus intra-GPU prefill/decode executor — Python host mirror.

This module mirrors the reference's library API (``nexussim``,
``/root/reference/proj/core/include/nexussim/*.hpp``) over the C-ABI of
``libnexus_b200.so`` (``include/nexus_b200.h``): the same names, argument
meanings and error behaviour (``ValueError`` where the reference throws
``std::invalid_argument``, ``RuntimeError`` for ``std::runtime_error``).
There is no Python or CPU fallback: if the library is missing, every call
raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

from . import _abi
from ._abi import (BatchMember, Breakdown, ControllerConfig, CostExt, DecodeCandidate, EngineConfig,
                   GpuSpec, KernelProfile, ModelConfig, OpWorkload, PartitionState, PhaseModel,
                   PrefillEntry, Request, SaturationCurve, SimConfig)
from ._abi import (NX_CLOCK_DEVICE, NX_CLOCK_REPLAY, NX_CLOCK_VIRTUAL, NX_ENGINE_MONOLITHIC,
                   NX_ENGINE_NEXUS, NX_ENGINE_STATIC, NX_MODE_DECODE, NX_MODE_PREFILL,
                   NX_PHASE_DECODE, NX_PHASE_PREFILL, NX_PREFILL_FCFS, NX_PREFILL_SPF)

__all__ = [
    "ModelConfig", "GpuSpec", "KernelProfile", "ControllerConfig", "EngineConfig", "SimConfig",
    "Request", "derive", "model_preset", "gpu_preset", "sim_config", "run", "Engine",
    "phase_latency_isolated", "decode_latency_contended", "compute_latency",
    "effective_decode_bandwidth", "prefill_batch_workloads", "decode_op_workloads",
    "mixed_batch_workloads", "select_mode", "adjust_partition", "PartitionController",
    "spf_schedule", "fcfs_prefill_schedule", "fcfs_decode_schedule", "chunked_mixed_schedule",
    "workload_trace", "trace_text", "parse_trace", "kernel_profile_text", "parse_kernel_profile",
]


def lib():
    return _abi.lib()


def _check(rc: int) -> int:
    if rc in (_abi.NX_OK, _abi.NX_EDONE, _abi.NX_EAGAIN):
        return rc
    msg = (lib().nx_last_error() or b"").decode()
    if rc == _abi.NX_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"nexus_b200 error {rc}: {msg}")


def _text(fn, *args) -> str:
    n = C.c_size_t(0)
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


# ---- presets (reference presets.cpp:13-29) --------------------------------

def derive(hidden_dim: int, ffn_dim: int, num_layers: int, num_heads: int,
           element_bytes: int = 2) -> ModelConfig:
    """ModelConfig::derive (domain.cpp:7-24)."""
    return lib().nx_model_derive(hidden_dim, ffn_dim, num_layers, num_heads, element_bytes)


_MODEL_PRESETS = {"tiny": (256, 1024, 8, 8, 2), "3b": (2048, 8192, 36, 16, 2),
                  "8b": (4096, 14336, 32, 32, 2), "14b": (5120, 13824, 48, 40, 2)}
_GPU_PRESETS = {"l20like": (92, 1.0e14, 8.64e11, 40 << 30), "desk": (64, 2.0e12, 1.0e11, 4 << 30),
                "desk-contention": (64, 2.0e13, 1.0e10, 8 << 30),
                "desk-tight": (64, 2.0e12, 1.0e11, 768 << 20)}


def model_preset(name: str) -> ModelConfig:
    return derive(*_MODEL_PRESETS[name])


def gpu_spec(total_sm: int, peak_compute: float, peak_bandwidth: float,
             kv_capacity_bytes: int) -> GpuSpec:
    g = GpuSpec()
    g.total_sm, g.peak_compute, g.peak_bandwidth = total_sm, peak_compute, peak_bandwidth
    g.kv_capacity_bytes = kv_capacity_bytes
    return g


def gpu_preset(name: str) -> GpuSpec:
    return gpu_spec(*_GPU_PRESETS[name])


def sim_config(model: ModelConfig, gpu: GpuSpec, *, kind: int = NX_ENGINE_NEXUS,
               static_r_p: int = 50, prefill_policy: int = NX_PREFILL_SPF,
               clock_mode: int = NX_CLOCK_VIRTUAL, ctrl: ControllerConfig | None = None,
               profile: KernelProfile | None = None, timeout_sim_s: float = 3600.0,
               max_events: int = 10_000_000, bw_sat: Sequence[float] | None = None,
               contention: Sequence[float] | None = None, decode_target_s: float = 0.0) -> SimConfig:
    """SimConfig; bw_sat (5 per-op shares) enables the SM-share-limited HBM
    bandwidth extension of the cost model (nx_cost_ext), None = reference;
    contention (c0, c1[, c2]) additionally replaces the contended-decode
    bandwidth split by the measured slowdown c0 + c1 p + c2 p^2 (p = the
    prefill lane's share); decode_target_s > 0 lets Algorithm 1's
    prefill-priority search also accept shares whose co-located decode step
    stays within that target (nx_cost_ext.decode_target_s)."""
    cfg = SimConfig()
    cfg.model = model
    cfg.gpu = gpu
    cfg.ctrl = ctrl if ctrl is not None else lib().nx_controller_config_default()
    cfg.profile = profile if profile is not None else lib().nx_kernel_profile_default()
    e = lib().nx_engine_config_default()
    e.kind, e.static_r_p, e.prefill_policy, e.clock_mode = kind, static_r_p, prefill_policy, clock_mode
    e.timeout_sim_s, e.max_events = timeout_sim_s, max_events
    cfg.engine = e
    if bw_sat is not None:
        cfg.ext = _ext(bw_sat, contention, decode_target_s)
    elif decode_target_s:
        raise ValueError("decode_target_s needs the cost-model extension (bw_sat)")
    return cfg


def _ext(bw_sat, contention=None, decode_target_s=0.0) -> CostExt:
    c = (0.0, 0.0, 0.0) if contention is None else tuple(contention) + (0.0,) * (3 - len(contention))
    return CostExt(1, 0 if contention is None else 1, (C.c_double * 5)(*bw_sat), (C.c_double * 3)(*c),
                   float(decode_target_s))


def set_cost_ext(bw_sat: Sequence[float] | None, contention: Sequence[float] | None = None) -> None:
    """Extension for the standalone cost-model calls (phase_latency_isolated, ...)."""
    if bw_sat is None:
        _check(lib().nx_set_cost_ext(None))
    else:
        _check(lib().nx_set_cost_ext(C.byref(_ext(bw_sat, contention))))


def validate_config(model, gpu, ctrl, prof) -> list[str]:
    buf = C.create_string_buffer(4096)
    n = lib().nx_validate_config(C.byref(model), C.byref(gpu), C.byref(ctrl), C.byref(prof), buf, 4096)
    return [] if n == 0 else buf.value.decode().split("; ")


# ---- operator / cost model -------------------------------------------------

def _ops_out():
    return (OpWorkload * _abi.NX_MAX_OPS)(), C.c_size_t(0)


def _i64(seq) -> C.Array:
    seq = list(seq)
    return (C.c_int64 * max(1, len(seq)))(*seq)


def prefill_batch_workloads(model: ModelConfig, chunks: Sequence[tuple[int, int]]) -> list[OpWorkload]:
    """prefill_batch_workloads (opcost.cpp:99-126); chunks are (tokens, context_len)."""
    out, n = _ops_out()
    _check(lib().nx_prefill_batch_workloads(C.byref(model), _i64(c[0] for c in chunks),
                                            _i64(c[1] for c in chunks), len(chunks), out, C.byref(n)))
    return list(out[: n.value])


def decode_op_workloads(model: ModelConfig, context_lens: Sequence[int]) -> list[OpWorkload]:
    out, n = _ops_out()
    _check(lib().nx_decode_op_workloads(C.byref(model), _i64(context_lens), len(context_lens), out,
                                        C.byref(n)))
    return list(out[: n.value])


def mixed_batch_workloads(model, chunks, decode_context_lens) -> list[OpWorkload]:
    out, n = _ops_out()
    _check(lib().nx_mixed_batch_workloads(C.byref(model), _i64(c[0] for c in chunks),
                                          _i64(c[1] for c in chunks), len(chunks),
                                          _i64(decode_context_lens), len(decode_context_lens),
                                          out, C.byref(n)))
    return list(out[: n.value])


def _ops_arr(ops: Sequence[OpWorkload]):
    return (OpWorkload * max(1, len(ops)))(*ops), len(ops)


def compute_latency(flops: float, share: float, curve: SaturationCurve, peak: float) -> float:
    out = C.c_double()
    _check(lib().nx_compute_latency(flops, share, curve, peak, C.byref(out)))
    return out.value


def phase_latency_isolated(ops, share, gpu, prof) -> Breakdown:
    arr, n = _ops_arr(ops)
    out = Breakdown()
    _check(lib().nx_phase_latency_isolated(arr, n, share, C.byref(gpu), C.byref(prof), C.byref(out)))
    return out


def decode_latency_contended(dops, share, prefill_bd, pops, gpu, prof) -> Breakdown:
    da, nd = _ops_arr(dops)
    pa, np_ = _ops_arr(pops)
    out = Breakdown()
    _check(lib().nx_decode_latency_contended(da, nd, share,
                                             C.byref(prefill_bd) if prefill_bd is not None else None,
                                             pa, np_, C.byref(gpu), C.byref(prof), C.byref(out)))
    return out


def effective_decode_bandwidth(p_attn, m_d, m_p1, m_p2, peak) -> float:
    out = C.c_double()
    _check(lib().nx_effective_decode_bandwidth(p_attn, m_d, m_p1, m_p2, peak, C.byref(out)))
    return out.value


def min_phase_latency(ops, gpu, prof) -> float:
    arr, n = _ops_arr(ops)
    return lib().nx_min_phase_latency(arr, n, C.byref(gpu), C.byref(prof))


# ---- controller ----------------------------------------------------------

def select_mode(kv_used: int, kv_capacity: int, kv_switch_fraction: float) -> int:
    m = lib().nx_select_mode(kv_used, kv_capacity, kv_switch_fraction)
    if m < 0:
        raise ValueError(lib().nx_last_error().decode())
    return m


class _Phase:
    """Keeps a Python latency callable alive behind an nx_phase_model."""

    def __init__(self, active: bool, fn: Callable[[int], float] | None):
        self._cb = _abi.LATENCY_FN(lambda _u, pct: float(fn(int(pct))) if fn else 0.0)
        self.pm = PhaseModel(1 if active else 0, self._cb, None)


def adjust_partition(target_phase: int, cur: PartitionState, prefill: tuple, decode: tuple,
                     cfg: ControllerConfig):
    """adjust_partition (optimizer.cpp:22-61); prefill/decode are (active, fn)."""
    p, d = _Phase(*prefill), _Phase(*decode)
    out = _abi.AdjustOutcome()
    _check(lib().nx_adjust_partition(target_phase, C.byref(cur), C.byref(p.pm), C.byref(d.pm),
                                     C.byref(cfg), C.byref(out)))
    return out


class PartitionController:
    """PartitionController (optimizer.hpp:60-77)."""

    def __init__(self, initial: PartitionState, cfg: ControllerConfig):
        self._h = C.c_void_p()
        _check(lib().nx_controller_create(C.byref(initial), C.byref(cfg), C.byref(self._h)))

    def decide(self, kv_used, kv_capacity, prefill: tuple, decode: tuple):
        p, d = _Phase(*prefill), _Phase(*decode)
        out = _abi.Decision()
        _check(lib().nx_controller_decide(self._h, kv_used, kv_capacity, C.byref(p.pm),
                                          C.byref(d.pm), C.byref(out)))
        return out

    def state(self) -> PartitionState:
        s = PartitionState()
        lib().nx_controller_state(self._h, C.byref(s))
        return s

    def __del__(self):
        if getattr(self, "_h", None):
            lib().nx_controller_destroy(self._h)
            self._h = None


# ---- schedulers ----------------------------------------------------------

def _entries(queue):
    q = list(queue)
    return (PrefillEntry * max(1, len(q)))(*[PrefillEntry(i, r, a) for (i, r, a) in q]), len(q)


def _cands(active):
    a = list(active)
    return (DecodeCandidate * max(1, len(a)))(*[DecodeCandidate(i, t) for (i, t) in a]), len(a)


def _plan(fn, *args, cap=4096):
    out = (BatchMember * cap)()
    n, tot = C.c_size_t(), C.c_int64()
    _check(fn(*args, out, cap, C.byref(n), C.byref(tot)))
    return [(m.id, m.tokens) for m in out[: n.value]], tot.value


def spf_schedule(queue, token_budget, gamma, now_s, skip_non_fitting=False):
    """spf_schedule (schedulers.cpp:43-64); queue = [(id, remaining, arrival_s)]."""
    q, n = _entries(queue)
    return _plan(lib().nx_spf_schedule, q, n, token_budget, gamma, now_s, int(skip_non_fitting))


def fcfs_prefill_schedule(queue, token_budget):
    q, n = _entries(queue)
    return _plan(lib().nx_fcfs_prefill_schedule, q, n, token_budget)


def fcfs_decode_schedule(active, max_batch):
    a, n = _cands(active)
    return _plan(lib().nx_fcfs_decode_schedule, a, n, max_batch)


def chunked_mixed_schedule(queue, active, token_budget, max_batch, chunk_size):
    q, nq = _entries(queue)
    a, na = _cands(active)
    return _plan(lib().nx_chunked_mixed_schedule, q, nq, a, na, token_budget, max_batch, chunk_size)


# ---- traces / calibration text ------------------------------------------

def workload_trace(preset: str, rate_rps: float, count: int, seed: int) -> list[Request]:
    """workload_preset + realize (presets.cpp:70-105)."""
    out = (Request * max(1, count))()
    n = C.c_size_t()
    _check(lib().nx_workload_preset_trace(preset.encode(), rate_rps, count, seed, out, count,
                                          C.byref(n)))
    return list(out[: n.value])


def trace_text(trace: Sequence[Request]) -> str:
    arr = (Request * max(1, len(trace)))(*trace)
    return _text(lib().nx_trace_to_text, arr, len(trace))


def parse_trace(text: str) -> list[Request]:
    cap = text.count("\n") + 1
    out = (Request * cap)()
    n = C.c_size_t()
    _check(lib().nx_trace_from_text(text.encode(), out, cap, C.byref(n)))
    return list(out[: n.value])


def kernel_profile_text(prof: KernelProfile) -> str:
    return _text(lib().nx_kernel_profile_to_text, C.byref(prof))


def parse_kernel_profile(text: str) -> tuple[KernelProfile, list[str]]:
    out = KernelProfile()
    w = C.create_string_buffer(4096)
    _check(lib().nx_kernel_profile_from_text(text.encode(), C.byref(out), w, 4096))
    return out, [x for x in w.value.decode().split("\n") if x]


# ---- engine ----------------------------------------------------------------

@dataclass
class SimResult:
    event_log: str
    decision_log: str
    summary_json: str
    stats: _abi.EngineStats
    requests: list = field(default_factory=list)
    timed_out: bool = False
    sim_end_s: float = 0.0


_LAUNCH_OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


def batch_from_desc(ptr) -> dict:
    """An nx_batch_desc (the device ABI's batch) as dict(lane, sm_pct,
    members=[dict(tokens, n, start, pages, sample)]); n is the member's token
    count, tokens are [] when the engine holds no token ids (no device bound)."""
    from ._dev_abi import BatchDesc
    d = C.cast(ptr, C.POINTER(BatchDesc)).contents
    members, t0, p0 = [], 0, 0
    for i in range(d.n_members):
        n, npg = d.n_tokens[i], d.n_pages[i]
        toks = [d.tokens[t0 + k] for k in range(n)] if d.tokens else []
        members.append(dict(tokens=toks, n=int(n), start=int(d.start_pos[i]),
                            pages=[d.pages[p0 + k] for k in range(npg)], sample=bool(d.sample[i])))
        t0 += n
        p0 += npg
    return dict(lane=int(d.lane), sm_pct=int(d.sm_pct), members=members)


class Engine:
    """The step executor (nx_engine_*): submit / step / run / logs / KV."""

    def __init__(self, cfg: SimConfig, device=None):
        self._h = C.c_void_p()
        self.cfg = cfg
        _check(lib().nx_engine_create(C.byref(cfg), C.byref(self._h)))
        self.device = None
        if device is not None:
            self.bind_device(device)

    def bind_device(self, device) -> None:
        _check(lib().nx_engine_bind_device(self._h, device.handle))
        self.device = device

    def _call(self, rc: int) -> int:
        if rc not in (_abi.NX_OK, _abi.NX_EDONE, _abi.NX_EAGAIN):
            msg = (lib().nx_engine_last_error(self._h) or b"").decode()
            if rc == _abi.NX_EINVAL:
                raise ValueError(msg)
            raise RuntimeError(f"nexus_b200 error {rc}: {msg}")
        return rc

    def submit(self, req: Request, tokens: Sequence[int] | None = None) -> None:
        if tokens is None:
            self._call(lib().nx_submit(self._h, C.byref(req)))
        else:
            arr = (C.c_int32 * len(tokens))(*tokens)
            self._call(lib().nx_submit_with_tokens(self._h, C.byref(req), arr))

    def submit_trace(self, trace: Sequence[Request]) -> None:
        arr = (Request * max(1, len(trace)))(*trace)
        self._call(lib().nx_submit_trace(self._h, arr, len(trace)))

    def step(self) -> int:
        rc = self._call(lib().nx_step(self._h))
        self._raise_observer_error()
        return rc

    def run(self) -> None:
        self._call(lib().nx_run(self._h))
        self._raise_observer_error()

    def set_replay_latencies(self, lat: Sequence[float]) -> None:
        arr = (C.c_double * max(1, len(lat)))(*lat)
        lib().nx_engine_set_replay_latencies(self._h, arr, len(lat))

    def set_logging(self, events: bool, pages: bool) -> None:
        lib().nx_engine_set_logging(self._h, int(events), int(pages))

    def set_slo(self, ttft_s: float, tbt_s: float) -> None:
        lib().nx_engine_set_slo(self._h, ttft_s, tbt_s)

    def set_launch_observer(self, fn: Callable[[dict], None] | None) -> None:
        """fn(batch) on every launch, before the device runs it (batch_from_desc
        form): rank 0 of an NX_TP_NCCL group forwards its batches to the
        followers with it (device.tp_follow). Exceptions inside fn cannot
        cross the C boundary; they are stored and re-raised by run()/step()."""
        if fn is None:
            self._obs = None
            _check(lib().nx_engine_set_launch_observer(self._h, None, None))
            return

        def cb(_user, ptr):
            try:
                fn(batch_from_desc(ptr))
            except BaseException as e:  # noqa: BLE001 -- surfaced after the C call returns
                self._obs_error = e

        self._obs_error = None
        self._obs = _LAUNCH_OBSERVER(cb)
        _check(lib().nx_engine_set_launch_observer(self._h, self._obs, None))

    def _raise_observer_error(self) -> None:
        e = getattr(self, "_obs_error", None)
        if e is not None:
            self._obs_error = None
            raise RuntimeError("launch observer failed") from e

    def configure_pages(self, page_tokens: int, num_pages: int) -> None:
        _check(lib().nx_kv_configure(self._h, page_tokens, num_pages))

    def stats(self) -> _abi.EngineStats:
        s = _abi.EngineStats()
        lib().nx_engine_get_stats(self._h, C.byref(s))
        return s

    def event_log(self) -> str:
        return _text(lib().nx_engine_event_log, self._h)

    def decision_log(self) -> str:
        return _text(lib().nx_engine_decision_log, self._h)

    def summary_json(self, label: str = "nexus") -> str:
        return _text(lib().nx_engine_summary_json, self._h, label.encode())

    def goodput(self) -> _abi.Goodput:
        g = _abi.Goodput()
        _check(lib().nx_engine_goodput(self._h, C.byref(g)))
        return g

    def _doubles(self, fn) -> list[float]:
        n = C.c_size_t()
        fn(self._h, None, 0, C.byref(n))
        out = (C.c_double * max(1, n.value))()
        fn(self._h, out, n.value, C.byref(n))
        return list(out[: n.value])

    def launch_latencies(self) -> list[float]:
        return self._doubles(lib().nx_engine_launch_latencies)

    def launch_device_ms(self) -> list[float]:
        return self._doubles(lib().nx_engine_launch_device_ms)

    def requests(self) -> list[_abi.RequestState]:
        n = C.c_size_t()
        lib().nx_engine_requests(self._h, None, 0, C.byref(n))
        out = (_abi.RequestState * max(1, n.value))()
        lib().nx_engine_requests(self._h, out, n.value, C.byref(n))
        return list(out[: n.value])

    def tokens(self, rid: int) -> list[int]:
        n = C.c_size_t()
        _check(lib().nx_engine_tokens(self._h, rid, None, 0, C.byref(n)))
        out = (C.c_int32 * max(1, n.value))()
        _check(lib().nx_engine_tokens(self._h, rid, out, n.value, C.byref(n)))
        return list(out[: n.value])

    def block_table(self, rid: int) -> list[int]:
        n = C.c_size_t()
        lib().nx_kv_block_table(self._h, rid, None, 0, C.byref(n))
        out = (C.c_int32 * max(1, n.value))()
        lib().nx_kv_block_table(self._h, rid, out, n.value, C.byref(n))
        return list(out[: n.value])

    def page_log(self) -> str:
        return _text(lib().nx_kv_page_log, self._h)

    def kv_usage(self) -> tuple[int, int, int]:
        u, r, c = C.c_int64(), C.c_int64(), C.c_int64()
        lib().nx_kv_usage(self._h, C.byref(u), C.byref(r), C.byref(c))
        return u.value, r.value, c.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().nx_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def run(cfg: SimConfig, trace: Sequence[Request]) -> SimResult:
    """nexus::run (simulator.cpp:760-770) for the intra-GPU engines."""
    eng = Engine(cfg)
    eng.submit_trace(trace)
    eng.run()
    st = eng.stats()
    label = {NX_ENGINE_NEXUS: "nexus", NX_ENGINE_STATIC: "static",
             NX_ENGINE_MONOLITHIC: "monolithic"}[cfg.engine.kind]
    res = SimResult(eng.event_log(), eng.decision_log(), eng.summary_json(label), st,
                    eng.requests(), bool(st.timed_out), st.clock_s)
    eng.close()
    return res

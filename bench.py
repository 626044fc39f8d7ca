#!/usr/bin/env python
"""Benchmark: SLO goodput of the Nexus executor on Llama-3.1-8B, one B200.

A *step* serves one fixed synthetic trace segment end to end: `--requests`
ShareGPT-shaped requests (reference presets.cpp:58-66 length fits) with
Poisson arrivals at `--rate` req/s, submitted through the C-ABI
(nx_submit_with_tokens: prompt ids from host buffers), executed by the
device-clock step executor (prefill and decode lanes on green-context SM
partitions, split chosen per launch by the cost model), with every sampled
token copied back to the host, then read out through nx_engine_tokens.

value  = SLO goodput on the engine clock: output tokens of requests with
         TTFT <= --slo-ttft and per-request p99 TBT <= --slo-tbt, per second of
         offered load (divided by the arrival window, first -> last arrival),
         summed over timed steps. (Dividing by the makespan instead measures
         the heavy-tailed longest output's decode time, not serving capacity;
         that number is reported as throughput_makespan.)
e2e    = the same good tokens divided by the client wall time of the whole
         call (submit from host buffers + serve + token read-back).
roofline = the dominant kernel class by device time (sampled CUDA-event
         pairs on the launching green-context stream), algorithmic bytes or
         FLOPs per launch / its event time, vs MEASURED_PEAKS.json.

`--impl reference` runs the reference's own CPU implementation of the path
(oracle/_ref: nexussim compiled from /root/reference) on the same trace and
config; it cannot execute a model, so its goodput is computed on its
cost-model clock with the B200 GpuSpec (reported with its CPU wall time).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# model -> (reference ModelConfig dims for the cost model (presets.cpp:13-19;
# 70B is derived the same way), real KV bytes/token of the kernel view).
MODELS = {
    "llama3-8b": ((4096, 14336, 32, 32, 2), 2 * 32 * 8 * 128 * 2),
    "qwen2.5-14b": ((5120, 13824, 48, 40, 2), 2 * 48 * 8 * 128 * 2),
    "llama3-70b": ((8192, 28672, 80, 64, 2), 2 * 80 * 8 * 128 * 2),
}


def ref_kvbpt(model: str) -> int:
    d, _, L, _, e = MODELS[model][0]
    return 2 * L * d * e


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=4)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="nexus", choices=["nexus", "reference"])
    p.add_argument("--engine", default="nexus", choices=["nexus", "static", "monolithic"])
    p.add_argument("--rate", type=float, default=128.0)
    p.add_argument("--requests", type=int, default=480)
    p.add_argument("--model", default="llama3-8b", choices=sorted(MODELS))
    p.add_argument("--workload", default="sharegpt",
                   help="trace preset: sharegpt | mixed | long-data | arxiv | longbench | bursty")
    p.add_argument("--kv-gb", type=float, default=80.0)
    p.add_argument("--slo-ttft", type=float, default=None,
                   help="TTFT SLO (s); default per model as frozen in BASELINE.md: 8B 1, 14B 4, 70B 2")
    p.add_argument("--slo-tbt", type=float, default=None,
                   help="per-request p99 TBT SLO (s); default 8B 0.05, 14B 0.075, 70B 0.1")
    p.add_argument("--profile-every", type=int, default=8)
    p.add_argument("--seed", type=int, default=101,
                   help="trace seed of the first step (seed + step per step). The controller knobs were swept "
                        "on seeds 1-24 (profiles/r01s2_*); 101+ are held out")
    p.add_argument("--static-r-p", type=int, default=50,
                   help="EngineConfig.static_r_p for --engine static (simulator.cpp:184-189)")
    p.add_argument("--compare", default="monolithic",
                   help="comma list of same-kernel baseline engines (monolithic, static) run on the identical "
                        "traces and prompts after the timed region; 'none' to skip")
    p.add_argument("--compare-steps", type=int, default=6,
                   help="baseline arm runs the first min(steps, this) timed traces (bounds the bench's wall "
                        "time); the ratios compare this engine on the same traces")
    p.add_argument("--no-green", action="store_true")
    p.add_argument("--calib", default=None,
                   help="calibration base path (.calib + .json from paper_2507_06608_b200.calibrate); "
                        "'none' = reference default profile and nominal B200 spec")
    p.add_argument("--no-bw-ext", action="store_true", help="disable the share-dependent bandwidth term")
    p.add_argument("--beta", type=float, default=1.5,
                   help="ControllerConfig.beta, the decode slack in prefill-prioritized mode (paper 1.1, set for "
                        "L20). 1.5 with decode batch 256 keeps decode steps short enough that a request's first "
                        "decode gap stays inside the TBT SLO (capacity 124 vs 119 rps for the monolithic "
                        "baseline on held-out seeds, profiles/r02_summary.md); 2.0 was round 1's default")
    p.add_argument("--gamma", type=float, default=None,
                   help="ControllerConfig.gamma (SPF aging, tokens of priority per second waited; reference "
                        "default 15). At 128 rps on B200 with the CTA-pair prefill GEMMs: gamma 15 -> 10145 tok/s "
                        "goodput, p99 TTFT 2.67 s; 1500 -> 10552, 1.03 s; 5000 -> 10669, 0.71 s "
                        "(profiles/r01s2_gamma_*.json). Default: 5000, except 15 for the long-prompt "
                        "longbench workload where shortest-prompt-first keeps more requests under the TTFT SLO "
                        "(C3: 152 vs 117 tok/s). The reference arm runs with the same gamma")
    p.add_argument("--decode-target-ms", type=float, default=0.0,
                   help="nx_cost_ext.decode_target_s (x 1e-3): in prefill-priority mode a prefill share also fits "
                        "when the decode batch's co-located step on the remaining SMs stays within this target, "
                        "so prefill takes every SM decode does not need (0 = the reference rule alone)")
    p.add_argument("--alpha", type=float, default=1.3, help="ControllerConfig.alpha (prefill slack, paper 1.3)")
    p.add_argument("--tp", type=int, default=0,
                   help="tensor-parallel group size (C4). 0 = auto: under torchrun with --model llama3-70b the "
                        "whole job is one TP group of WORLD_SIZE GPUs driven by rank 0 (NX_TP_PEER: our peer-memory "
                        "all-reduce kernels over NVLink, one engine, device clock); otherwise 1")
    p.add_argument("--tp-mode", default="peer", choices=["peer", "nccl"],
                   help="peer: rank 0 drives every GPU of the group (our peer-memory collectives); nccl: one "
                        "process per GPU with NCCL all-reduces, rank 0's engine forwarding every launch to the "
                        "followers (device.tp_follow) so all ranks run identical batches on its device clock")
    p.add_argument("--tp-colocated", action="store_true",
                   help="place all TP ranks on one GPU (NX_TP_PEER_COLOCATED; a functional check of the TP path)")
    p.add_argument("--token-budget", type=int, default=4096,
                   help="ControllerConfig.token_budget: prompt tokens per prefill batch of this engine (and "
                        "chunk_size when --engine monolithic). 4096: nexus' prefill lane runs at saturation at "
                        "the bench rate, so batch efficiency is capacity (profiles/r02_summary.md)")
    p.add_argument("--compare-token-budget", type=int, default=2048,
                   help="token budget / chunk of the same-kernel baseline arm: 2048 is the monolithic engine's "
                        "best (3072 and 4096 lower its capacity: its TBT grows with the chunk)")
    p.add_argument("--max-decode-batch", type=int, default=256,
                   help="ControllerConfig.max_decode_batch (reference default 64, domain.hpp:87)")
    return p.parse_args()


def partition_roofline(dom, c, pk):
    sms = c.get("mean_partition_sms", 0.0)
    if not sms:
        return None
    mhz = pk.get("sm_max_mhz", 1965.0)
    if dom in ("gemm_prefill", "attn_prefill"):
        ceil = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) * sms / 148.0
        return {"mean_sms": sms, "ceiling": ceil, "unit": "TFLOP/s", "frac": c["TFLOPs"] / ceil,
                "ceiling_rule": "sustained bf16 peak x mean SMs / 148"}
    if dom == "gemm_decode":
        ceil = min(pk["hbm_gbs"], sms * 64 * mhz * 1e6 / 1e9)
        return {"mean_sms": sms, "ceiling": ceil, "unit": "GB/s", "frac": c["GBps"] / ceil,
                "ceiling_rule": "min(HBM peak, mean SMs x 64 B/cycle x max SM clock)"}
    ceil = pk["hbm_gbs"] * min(1.0, sms / 148.0 * 2.0)
    return {"mean_sms": sms, "ceiling": ceil, "unit": "GB/s", "frac": c["GBps"] / ceil,
            "ceiling_rule": "HBM peak (reachable from ~half the SMs)"}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---- metrics from a reference-format event log (same code for both arms) --

def log_metrics(event_log: str, slo_ttft: float, slo_tbt: float):
    arrival, times, finish = {}, {}, {}
    for line in event_log.splitlines():
        c = line.split("\t")
        t, kind, members = float(c[0]), c[2], c[3]
        if members == "-":
            continue
        for m in members.split(","):
            rid, _tok, emitted = (int(x) for x in m.split(":"))
            if kind == "arrival":
                arrival[rid] = t
            elif kind == "complete" and emitted:
                times.setdefault(rid, []).extend([t] * emitted)
            elif kind == "finish":
                finish[rid] = t
    ttft, gaps_all, good, out_tokens, good_reqs = [], [], 0, 0, 0
    for rid, f in finish.items():
        ts = times[rid]
        tt = ts[0] - arrival[rid]
        gaps = [b - a for a, b in zip(ts, ts[1:])]
        ttft.append(tt)
        gaps_all.extend(gaps)
        out_tokens += len(ts)
        p99 = sorted(gaps)[max(0, -(-99 * len(gaps) // 100) - 1)] if gaps else 0.0
        if tt <= slo_ttft and p99 <= slo_tbt:
            good += len(ts)
            good_reqs += 1
    span = (max(finish.values()) - min(arrival.values())) if finish else 0.0
    window = (max(arrival.values()) - min(arrival.values())) if arrival else 0.0
    return dict(good_tokens=good, out_tokens=out_tokens, makespan=span, window=window, ttft=ttft,
                tbt=gaps_all, completed=len(finish), good_requests=good_reqs)


def nearest_rank(v, p):
    """Nearest-rank percentile (reference metrics.cpp:30-38)."""
    if not v:
        return 0.0
    v = sorted(v)
    import math
    k = min(len(v), max(1, math.ceil(p / 100.0 * len(v))))
    return v[k - 1]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.rows, self.proc, self.gpu = [], None, gpu_index

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sms = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        loaded = sorted(sms)
        return {"sm_mhz": loaded[len(loaded) // 2] if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # scalar barrier / max only; no data-path collective
        return rank, world, local, dist
    return rank, world, local, None


def load_calib(base):
    """(peak_compute, peak_bandwidth, profile, bw_sat, contention (c0, c1) or
    None) from a calibration, or None."""
    if not base or base == "none" or not os.path.exists(base + ".json"):
        return None
    import paper_2507_06608_b200 as nx
    d = json.load(open(base + ".json"))
    prof, _ = nx.parse_kernel_profile(open(base + ".calib").read())
    cf = d.get("contention_fit")
    return (d["gpu_spec"]["peak_compute"], d["gpu_spec"]["peak_bandwidth"], prof, d["bw_sat"],
            (cf["c0"], cf["c1"], cf.get("c2", 0.0)) if cf else None)


def make_cfg(nx, engine, num_pages, page_tokens, clock_mode, calib, bw_ext=True, max_decode_batch=64,
             alpha=1.3, beta=1.1, model="llama3-8b", gamma=None, static_r_p=50, tp=1, token_budget=2048,
             decode_target_s=0.0):
    """tp > 1: the GpuSpec describes the TP group (peaks x tp; every GPU holds
    its kv heads of the same token pages, so the token capacity is one GPU's)."""
    m = nx.derive(*MODELS[model][0])
    slack = 4096
    cap_tokens = (num_pages - slack) * page_tokens
    cal = load_calib(calib)
    C, B, prof, bw_sat, cont = (1.6595e15, 6.5562e12, None, None, None) if cal is None else cal
    g = nx.gpu_spec(148, C * tp, B * tp, cap_tokens * ref_kvbpt(model))
    kind = {"nexus": nx.NX_ENGINE_NEXUS, "static": nx.NX_ENGINE_STATIC,
            "monolithic": nx.NX_ENGINE_MONOLITHIC}[engine]
    ctrl = nx.lib().nx_controller_config_default()
    ctrl.max_decode_batch = max_decode_batch
    ctrl.token_budget = ctrl.chunk_size = token_budget
    ctrl.alpha, ctrl.beta = alpha, beta
    if gamma is not None:
        ctrl.gamma = gamma
    return nx.sim_config(m, g, kind=kind, clock_mode=clock_mode, profile=prof, ctrl=ctrl,
                         bw_sat=bw_sat if bw_ext else None, static_r_p=static_r_p,
                         contention=cont if bw_ext else None,
                         decode_target_s=decode_target_s if bw_ext and bw_sat is not None else 0.0)


def reference_cfg(args, num_pages, page_tokens, engine=None):
    """SimConfig for the reference arm built through the reference library
    alone (oracle/_ref: ModelConfig::derive, default-constructed configs,
    load_kernel_profile presets.cpp:128-170); libnexus_b200.so is never
    loaded in this process."""
    from oracle import reference
    from paper_2507_06608_b200 import _abi  # POD struct layouts only; loads no library
    m = reference.model_derive(*MODELS[args.model][0])
    g = _abi.GpuSpec()
    g.total_sm, g.peak_compute, g.peak_bandwidth = 148, 1.6595e15, 6.5562e12
    prof = None
    if args.calib and args.calib != "none" and os.path.exists(args.calib + ".json"):
        d = json.load(open(args.calib + ".json"))
        g.peak_compute, g.peak_bandwidth = d["gpu_spec"]["peak_compute"], d["gpu_spec"]["peak_bandwidth"]
        prof, _ = reference.load_kernel_profile_text(open(args.calib + ".calib").read())
    g.kv_capacity_bytes = (num_pages - 4096) * page_tokens * ref_kvbpt(args.model)
    ctrl, _, _ = reference.defaults()
    ctrl.max_decode_batch, ctrl.alpha, ctrl.beta = args.max_decode_batch, args.alpha, args.beta
    ctrl.token_budget = ctrl.chunk_size = args.token_budget
    if args.gamma is not None:
        ctrl.gamma = args.gamma
    kind = {"nexus": _abi.NX_ENGINE_NEXUS, "static": _abi.NX_ENGINE_STATIC,
            "monolithic": _abi.NX_ENGINE_MONOLITHIC}[engine or args.engine]
    return reference.sim_config(m, g, kind=kind, static_r_p=args.static_r_p, ctrl=ctrl, profile=prof)


def run_reference(args, rank, world, dist):
    """The reference's CPU implementation (oracle/_ref: nexussim compiled from
    /root/reference), same trace generator (workload.cpp presets), same model,
    calibration and controller settings; its goodput is computed on its own
    cost-model clock. Only rank 0 runs it."""
    if rank != 0:
        return
    from oracle import reference
    if not reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libnexussim_ref.so not built"}))
        return
    if args.workload not in ("sharegpt", "mixed", "long-data", "arxiv"):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"workload {args.workload!r} is not a reference preset (presets.cpp:58-90)"}))
        return
    page_tokens = 16
    num_pages = int(args.kv_gb * (1 << 30) // (page_tokens * MODELS[args.model][1]))
    cfg = reference_cfg(args, num_pages, page_tokens)
    good = span = window = out = wall = 0.0
    ttft, tbt, decisions = [], [], 0
    for step in range(args.warmup + args.steps):
        trace = reference.workload_trace(args.workload, args.rate, args.requests, args.seed + step)
        t0 = time.perf_counter()
        r = reference.run(cfg, trace)
        t1 = time.perf_counter()
        if step < args.warmup:
            continue
        m = log_metrics(r["event_log"], args.slo_ttft, args.slo_tbt)
        good += m["good_tokens"]
        span += m["makespan"]
        window += m["window"]
        out += m["out_tokens"]
        wall += t1 - t0
        ttft += m["ttft"]
        tbt += m["tbt"]
        decisions += r["decision_log"].count("\n") - 1
    value = good / window if window else 0.0
    loaded = sorted({os.path.basename(l.split()[-1]) for l in open("/proc/self/maps")
                     if l.rstrip().endswith(".so") and ("nexus" in l)})
    line = {
        "impl": "reference", "metric": "goodput_tok_per_s_at_slo",
        "slo_attainment": good / out if out else 0.0, "throughput_makespan": out / span if span else 0.0,
        "value": value, "unit": "tok/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * wall / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.model} (reference cost-model preset), {args.workload} trace",
                   "rate_rps": args.rate,
                   "requests_per_step": args.requests, "engine": args.engine, "seed": args.seed,
                   "slo": {"ttft_s": args.slo_ttft, "tbt_p99_s": args.slo_tbt}},
        "ttft_p50": nearest_rank(ttft, 50), "ttft_p99": nearest_rank(ttft, 99),
        "tbt_p50": nearest_rank(tbt, 50), "tbt_p99": nearest_rank(tbt, 99),
        "libraries_loaded": loaded,
        "cpu_baseline": {"value": value, "unit": "tok/s", "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} x {args.requests} {args.workload} requests on nexussim's cost-model "
                                   f"clock (predicted, not executed); CPU wall {wall:.3f}s, "
                                   f"{1e6 * wall / max(1, decisions):.2f} us/decision"},
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    args = parse()
    slo = {"llama3-8b": (1.0, 0.05), "qwen2.5-14b": (4.0, 0.075), "llama3-70b": (2.0, 0.1)}[args.model]
    args.slo_ttft = slo[0] if args.slo_ttft is None else args.slo_ttft
    args.slo_tbt = slo[1] if args.slo_tbt is None else args.slo_tbt
    if args.gamma is None:
        args.gamma = 15.0 if args.workload == "longbench" else 5000.0
    if args.calib is None:
        args.calib = os.path.join(REPO, "profiles", "b200_" + args.model.replace(".", "_").replace("-", "_"))
    rank, world, local, dist = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, world, dist)
        return
    tp = args.tp or (world if args.model == "llama3-70b" and world > 1 else 1)
    tp_nccl = tp > 1 and args.tp_mode == "nccl"
    if tp_nccl and tp != world:
        raise SystemExit(f"--tp-mode nccl needs one process per rank: --tp {tp} != WORLD_SIZE {world}")
    if tp > 1 and world > 1 and not tp_nccl:
        # one TP group over all GPUs of the job, driven by rank 0 (one engine,
        # one device clock); the other ranks only hold the barriers
        if tp != world:
            raise SystemExit(f"--tp {tp} must equal WORLD_SIZE {world} under torchrun")
        if rank != 0:
            dist.barrier()
            dist.barrier()
            return
    import numpy as np
    import paper_2507_06608_b200 as nx
    from paper_2507_06608_b200 import device as D

    page_tokens = 16
    num_pages = int(args.kv_gb * (1 << 30) * tp // (page_tokens * MODELS[args.model][1]))
    dev_kw = dict(num_pages=num_pages, page_tokens=page_tokens,
                  max_prefill_tokens=max(args.token_budget, args.compare_token_budget) + args.max_decode_batch,
                  max_decode_batch=args.max_decode_batch, seed=args.seed)
    if tp_nccl:
        # one communicator per lane; ids from rank 0, every rank holds its shard
        box = [[D.nccl_unique_id(), D.nccl_unique_id()] if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        dev = D.Device(D.arch_preset(args.model), green_contexts=not args.no_green, device=local, tp_size=tp,
                       tp_rank=rank, tp_mode=D.NX_TP_NCCL, nccl_ids=box[0], **dev_kw)
        if rank != 0:
            def recv():
                b = [None]
                dist.broadcast_object_list(b, src=0)
                return b[0]
            D.tp_follow(dev, recv)
            dev.close()
            return
    else:
        tp_mode = D.NX_TP_PEER_COLOCATED if args.tp_colocated else D.NX_TP_PEER
        dev = D.Device(D.arch_preset(args.model), green_contexts=not args.no_green and not (tp > 1 and args.tp_colocated),
                       device=0 if tp > 1 else local, **(dict(tp_size=tp, tp_mode=tp_mode) if tp > 1 else {}),
                       **dev_kw)
    try:
        run_bench(args, rank, world, local, dist, nx, D, np, dev, tp, tp_nccl, num_pages, page_tokens)
    finally:
        if tp_nccl:
            dist.broadcast_object_list([None], src=0)  # followers leave tp_follow


def run_bench(args, rank, world, local, dist, nx, D, np, dev, tp, tp_nccl, num_pages, page_tokens):
    dev.set_profiling(args.profile_every)
    group_world = 1 if tp > 1 else world  # ranks whose results are aggregated

    def cfg_for(engine, token_budget=None):
        return make_cfg(nx, engine, num_pages, page_tokens, nx.NX_CLOCK_DEVICE, args.calib, not args.no_bw_ext,
                        args.max_decode_batch, args.alpha, args.beta, args.model, args.gamma, args.static_r_p, tp,
                        token_budget or args.token_budget, args.decode_target_ms / 1e3)

    cfg = cfg_for(args.engine)
    vocab = dev.arch.vocab
    rng = np.random.default_rng(args.seed + 7919 * rank)
    inputs = {}

    def step_inputs(step):
        """The step's trace and prompt ids (host buffers), fixed per step so the
        same-kernel baseline engines see identical inputs."""
        if step not in inputs:
            trace = nx.workload_trace(args.workload, args.rate, args.requests, args.seed + step + 1000 * rank)
            inputs[step] = (trace, [rng.integers(0, vocab, t.prompt_len, dtype=np.int32) for t in trace])
        return inputs[step]

    def one_step(step, scfg=None):
        trace, prompts = step_inputs(step)
        t0 = time.perf_counter()
        eng = nx.Engine(scfg or cfg, device=dev)
        if tp_nccl:
            eng.set_launch_observer(lambda b: dist.broadcast_object_list([b], src=0))
        eng.set_slo(args.slo_ttft, args.slo_tbt)
        eng.set_logging(True, False)
        for t, p in zip(trace, prompts):
            eng.submit(t, p.tolist())
        eng.run()
        toks = [eng.tokens(t.id) for t in trace]
        t1 = time.perf_counter()
        m = log_metrics(eng.event_log(), args.slo_ttft, args.slo_tbt)
        m["wall"] = t1 - t0
        m["launches"] = eng.stats().launches
        m["h2d"] = sum(4 * t.prompt_len for t in trace)
        m["d2h"] = 4 * sum(len(x) - t.prompt_len for x, t in zip(toks, trace))
        dlog = eng.decision_log()
        m["decisions"] = dlog.count("\n") - 1
        m["switches"] = eng.stats().switches
        # applied prefill share of the decisions taken while requests arrive
        t_end = trace[-1].arrival_s
        hist = {}
        for line in dlog.splitlines()[1:]:
            f = line.split("\t")
            if float(f[0]) <= t_end:
                hist[int(f[4])] = hist.get(int(f[4]), 0) + 1
        m["r_p_hist"] = hist
        eng.close()
        return m

    for s in range(args.warmup):
        one_step(s)
    dev.reset_kernel_stats()
    k0 = dev.kernel_stats().kernel_launches
    clocks = ClockSampler(local)
    if dist and not tp_nccl:  # (NCCL followers are inside tp_follow, in lockstep through the collectives)
        dist.barrier()
    clocks.start()
    results = [one_step(args.warmup + s) for s in range(args.steps)]
    clk = clocks.stop()
    ks = dev.kernel_stats()
    good = sum(r["good_tokens"] for r in results)
    out_tok = sum(r["out_tokens"] for r in results)
    span = sum(r["makespan"] for r in results)
    window = sum(r["window"] for r in results)
    wall = sum(r["wall"] for r in results)
    if dist and tp > 1 and not tp_nccl:
        dist.barrier()
    if dist and tp == 1:
        import torch
        t = torch.tensor([good, out_tok, span, window], dtype=torch.float64)
        w = torch.tensor([wall, window], dtype=torch.float64)
        dist.all_reduce(t)  # sum over ranks
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        good, out_tok, span_sum, window_sum = t.tolist()
        wall_max, window_max = w.tolist()
    else:
        span_sum, window_sum, wall_max, window_max = span, window, wall, window
    # whole-job good tokens per second of offered load (max window over ranks)
    value = good / window_max if window_max else 0.0
    # client view: the same good tokens over the wall time of submit + serve +
    # read-back, restricted to the arrival window share of that wall time
    e2e = good / (wall_max * window_max / (span_sum / group_world)) if wall_max and span_sum else 0.0
    ttft = [x for r in results for x in r["ttft"]]
    tbt = [x for r in results for x in r["tbt"]]

    def summarize(rs):
        g = sum(r["good_tokens"] for r in rs)
        o = sum(r["out_tokens"] for r in rs)
        w = sum(r["window"] for r in rs)
        sp = sum(r["makespan"] for r in rs)
        tt = [x for r in rs for x in r["ttft"]]
        tb = [x for r in rs for x in r["tbt"]]
        return {"goodput": g / w if w else 0.0, "goodput_makespan": g / sp if sp else 0.0,
                "slo_attainment": g / o if o else 0.0, "throughput_makespan": o / sp if sp else 0.0,
                "ttft_p50": nearest_rank(tt, 50), "ttft_p99": nearest_rank(tt, 99),
                "tbt_p50": nearest_rank(tb, 50), "tbt_p99": nearest_rank(tb, 99),
                "ms_per_step": 1000 * sum(r["wall"] for r in rs) / max(1, len(rs))}

    # Same-kernel baselines (BASELINE.md §2 / SURVEY §8(f)1): the identical traces
    # and prompt buffers served by the monolithic chunked-prefill engine (and/or
    # a static split), after the timed region so `value` times this engine only.
    n_cmp = max(1, min(args.steps, args.compare_steps))
    mine = summarize(results[:n_cmp])
    baselines = {}
    for bname in [e.strip() for e in args.compare.split(",")]:
        if not bname or bname == "none" or bname == args.engine:
            continue
        b = summarize([one_step(args.warmup + s, cfg_for(bname, args.compare_token_budget)) for s in range(n_cmp)])
        b["traces"] = f"the first {n_cmp} timed traces"
        b["token_budget"] = args.compare_token_budget
        b["this_engine_same_traces"] = mine
        b["this_engine_over_baseline"] = {
            "goodput": mine["goodput"] / b["goodput"] if b["goodput"] else None,
            "goodput_makespan": mine["goodput_makespan"] / b["goodput_makespan"] if b["goodput_makespan"] else None,
            "ttft_p99": mine["ttft_p99"] / b["ttft_p99"] if b["ttft_p99"] else None,
            "tbt_p99": mine["tbt_p99"] / b["tbt_p99"] if b["tbt_p99"] else None}
        baselines[bname if bname != "static" else f"static_r_p{args.static_r_p}"] = b
    pk, pk_kind = peaks()
    names = ["gemm_decode", "gemm_prefill", "attn_decode", "attn_prefill", "other"]
    classes = {}
    for i, n in enumerate(names):
        if ks.launches[i]:
            per_ms = ks.ms[i] / ks.launches[i]
            classes[n] = {"ms_total_sampled": ks.ms[i], "launches_sampled": ks.launches[i],
                          "GBps": ks.bytes[i] / ks.ms[i] / 1e6 if ks.ms[i] else 0.0,
                          "TFLOPs": ks.flops[i] / ks.ms[i] / 1e9 if ks.ms[i] else 0.0,
                          "avg_launch_ms": per_ms,
                          "mean_partition_sms": ks.sm_ms[i] / ks.ms[i] if ks.ms[i] else 0.0}
    dom = max(classes, key=lambda n: classes[n]["ms_total_sampled"]) if classes else None
    roof = None
    if dom:
        c = classes[dom]
        i = names.index(dom)
        tensor = dom in ("gemm_prefill", "attn_prefill")
        if tensor:
            ach, peak, unit = c["TFLOPs"], pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), "TFLOP/s"
        else:
            ach, peak, unit = c["GBps"], pk["hbm_gbs"], "GB/s"
        alg_bytes = ks.bytes[i] / ks.launches[i]
        traffic, traffic_src = None, None
        try:  # DRAM bytes / algorithmic bytes of this kernel class from one ncu --set full capture
            with open(os.path.join(REPO, "profiles", "dram_traffic.json")) as f:
                t = json.load(f).get(dom)
            if t:
                traffic, traffic_src = t["dram_over_algorithmic"] * alg_bytes, t["source"]
        except (OSError, ValueError):
            pass
        roof = {"bound": "tensor" if tensor else "hbm", "kernel_class": dom, "achieved": ach, "peak": peak,
                "peak_source": pk_kind + (" sustained" if tensor else ""), "unit": unit,
                "frac": ach / peak if peak else None,
                "traffic": traffic, "traffic_unit": "bytes per launch", "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": alg_bytes,
                "algorithmic_per_launch": (ks.flops[i] if tensor else ks.bytes[i]) / ks.launches[i],
                # the launches ran on green-context partitions: the HBM peak is not
                # reachable by a decode GEMM on a few dozen SMs, whose per-SM ceiling
                # is 64 B of weights per cycle (tcgen05 M = 128 floor, profiles/r01s2_mma_probe.md)
                "partition": partition_roofline(dom, c, pk),
                "share_of_sampled_device_time": ks.ms[i] / ks.batch_ms_sampled if ks.batch_ms_sampled else None}
    if rank != 0:
        return
    cpu = None
    try:
        from oracle import reference
        if reference.available():
            tr = reference.workload_trace(args.workload, args.rate, args.requests, args.seed + args.warmup)
            t0 = time.perf_counter()
            rr = reference.run(reference_cfg(args, num_pages, page_tokens), tr)
            cw = time.perf_counter() - t0
            mm = log_metrics(rr["event_log"], args.slo_ttft, args.slo_tbt)
            cpu = {"value": mm["good_tokens"] / mm["window"] if mm["window"] else 0.0, "unit": "tok/s",
                   "cores": 1, "kind": "reference",
                   "sample": f"the first timed step's trace ({args.requests} {args.workload} requests) through "
                             f"nexussim (oracle/_ref) on its cost-model clock with the calibrated B200 spec "
                             f"(predicted goodput, not executed); CPU wall {cw:.3f}s"}
    except Exception as e:  # the baseline is reported, never required
        cpu = {"unavailable": str(e)}
    line = {
        "metric": "goodput_tok_per_s_at_slo", "value": value, "unit": "tok/s",
        "n_gpus": world if tp == 1 else (1 if args.tp_colocated else tp),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * wall_max / args.steps,
        "higher_is_better": True, "scaling": "strong" if tp > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, sharegpt-shaped lengths, random prompt ids)",
        "config": {"workload": f"{args.model} bf16, " + (f"TP={tp} group" if tp > 1 else "1 B200 per rank") + f", {args.workload} trace"
                               + (" (BASELINE configs[1])" if args.model == "llama3-8b" and args.workload == "sharegpt" else ""),
                   "rate_rps": args.rate, "requests_per_step": args.requests, "engine": args.engine,
                   "seed": args.seed, "static_r_p": args.static_r_p if args.engine == "static" else None,
                   "clock": "device", "green_contexts": not args.no_green,
                   "calibration": os.path.basename(args.calib) if load_calib(args.calib) else "none",
                   "bw_ext": not args.no_bw_ext,
                   "slo": {"ttft_s": args.slo_ttft, "tbt_p99_s": args.slo_tbt},
                   "max_decode_batch": args.max_decode_batch, "token_budget": args.token_budget,
                   "alpha": args.alpha, "beta": args.beta, "gamma": args.gamma,
                   "decode_target_ms": args.decode_target_ms,
                   "kv_pool_gb": args.kv_gb,
                   "parallelism": (f"tp{tp}" + (" colocated on one GPU" if args.tp_colocated
                                                else " (NCCL all-reduce, one process per GPU)" if tp_nccl
                                                else " (peer-memory all-reduce)"))
                   if tp > 1 else f"replicas x{world}",
                   "l2": "inputs > L2 (16 GB weights streamed per decode step)"},
        "ttft_p50": nearest_rank(ttft, 50), "ttft_p99": nearest_rank(ttft, 99),
        "tbt_p50": nearest_rank(tbt, 50), "tbt_p99": nearest_rank(tbt, 99),
        "completed": sum(r["completed"] for r in results), "good_tokens": good,
        "output_tokens": out_tok, "slo_attainment": good / out_tok if out_tok else 0.0,
        "throughput_makespan": out_tok / (span_sum / group_world) if span_sum else 0.0,
        "goodput_makespan": good / (span_sum / group_world) if span_sum else 0.0,
        "same_kernel_baselines": baselines,
        # not measured in this run: the paper's throughput metric from tools/capacity.py (3 held-out seeds x
        # 2,000 requests per probe, >= 90% of requests inside both SLOs), same defaults as this line
        "capacity_rps_reference": {"source": ["profiles/r02_capacity_8b_refit_seeds301.json",
                                              "profiles/r02_capacity_8b_mono_page_seeds301.json"],
                                   "nexus": 124.0, "monolithic": 119.0} if args.model == "llama3-8b" else None,
        "decisions": sum(r["decisions"] for r in results), "switches": sum(r["switches"] for r in results),
        "r_p_hist_arrivals": {str(k): sum(r["r_p_hist"].get(k, 0) for r in results)
                              for k in sorted({k for r in results for k in r["r_p_hist"]})},
        "e2e": {"value": e2e, "unit": "tok/s", "h2d_bytes_per_step": sum(r["h2d"] for r in results) // args.steps,
                "d2h_bytes_per_step": sum(r["d2h"] for r in results) // args.steps},
        "gpu_launches": int(ks.kernel_launches - k0),
        "roofline": roof, "kernel_classes": classes, "clocks": clk, "cpu_baseline": cpu,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()

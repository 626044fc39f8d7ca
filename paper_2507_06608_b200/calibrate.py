"""On-device profiler -> cost-model calibration.

Measures, on the real B200 partitions, the latency of a representative
prefill batch and decode batch of the served model on every pre-instantiated
green-context layout (the diminishing-returns curves of PAPER.md:462-464),
plus decode latency alone vs co-located with a prefill batch (the contention
the cost model's B_decode term predicts). It then refits the
cost model so its predictions match the device:

  * GpuSpec.peak_compute / peak_bandwidth := effective full-GPU rates;
  * per-operator (r_sat, lambda) of Eq. 5: QKV, prefill attention, O and FFN
    each from their own sampled share of the prefill sweep (kernel event
    pairs charged to their reference operator, nx_kernel_stats.op_ms);
  * per-operator bw_sat of the flagged bandwidth extension (nx_cost_ext)
    from the decode sweep, likewise per operator (decode attention's memory
    term carries its calibration: its compute curve never binds);
  * the measured co-location slowdown c0 + c1 p + c2 p^2 (p = prefill share)
    (nx_cost_ext.contention) from the co-located decode sweep.

Outputs the reference calibration file format (presets.cpp:109-170,
"<op> <r_sat> <lambda>") and a JSON with the spec, bw_sat and raw data.

    python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b
"""
from __future__ import annotations

import argparse
import json
import math
import statistics
import time

import numpy as np

import paper_2507_06608_b200 as nx
from paper_2507_06608_b200 import device as D


OPS = ("qkv_proj", "attn_prefill", "attn_decode", "attn_out_proj", "ffn")  # NX_OP_* order


def measure(dev, members, lane, pct, reps=5, warm=2):
    """Median batch time (ms, unprofiled) and the per-operator split of one
    batch (ms; sampled CUDA-event pairs per kernel charged to their reference
    operator, nx_kernel_stats.op_ms, rescaled to the unprofiled total)."""
    for _ in range(warm):
        dev.forward(members, lane=lane, sm_pct=pct)
    ts = [dev.forward(members, lane=lane, sm_pct=pct)[2] for _ in range(reps)]
    dev.set_profiling(1)
    dev.reset_kernel_stats()
    for _ in range(reps):
        dev.forward(members, lane=lane, sm_pct=pct)
    ks = dev.kernel_stats()
    dev.set_profiling(0)
    total = statistics.median(ts)
    ops = [ks.op_ms[k] / reps for k in range(5)]
    scale = total / sum(ops) if sum(ops) > 0 else 0.0
    return total, [o * scale for o in ops]


def op_sums(ops, field):
    out = [0.0] * 5
    for o in ops:
        out[o.kind] += getattr(o, field)
    return out


def _shape_err(model_s, times_ms):
    """Log-space error after the best common scale: fits the curve's shape only
    (one cost model peak serves every operator, so per-operator levels are not
    representable; the phase fit sets the level)."""
    d = [math.log(m) - math.log(t * 1e-3) for m, t in zip(model_s, times_ms)]
    mu = statistics.mean(d)
    return sum((x - mu) ** 2 for x in d)


def fit_curve(flops, shares, times_ms, C):
    """Shape of one operator's Eq. 5 curve: (r_sat, lambda), r_sat in (0, 1]."""
    best = None
    for i in range(5, 101):
        r_sat = i / 100.0
        for j in range(0, 101):
            lam = j / 50.0
            m = [flops * (1.0 / s if s <= r_sat else (1.0 / r_sat) * (1.0 + lam * (s - r_sat))) / C for s in shares]
            err = _shape_err(m, times_ms)
            if best is None or err < best[0] - 1e-15:
                best = (err, r_sat, lam)
    return {"r_sat": best[1], "lambda": best[2], "rms_log_err_shape": math.sqrt(best[0] / len(shares))}


def fit_bw_sat(mem, shares, times_ms, B):
    """Shape of one operator's share-limited memory term (nx_cost_ext bw_sat)."""
    best = None
    for i in range(2, 101):
        sat = i / 100.0
        err = _shape_err([mem / (B * min(1.0, s / sat)) for s in shares], times_ms)
        if best is None or err < best[0] - 1e-15:
            best = (err, sat)
    return {"bw_sat": best[1], "rms_log_err_shape": math.sqrt(best[0] / len(shares))}


def fit_contention(points):
    """Least squares slowdown = c0 + c1 p + c2 p^2 over the co-location sweep
    (p = the prefill lane's share of the SMs)."""
    x = np.array([p["prefill_sms"] / (p["prefill_sms"] + p["decode_sms"]) for p in points])
    y = np.array([p["slowdown"] for p in points])
    A = np.stack([np.ones_like(x), x, x * x], 1)
    c, *_ = np.linalg.lstsq(A, y, rcond=None)
    pred = A @ c
    return {"c0": float(c[0]), "c1": float(c[1]), "c2": float(c[2]),
            "max_rel_err": float(np.max(np.abs(pred / y - 1.0)))}


def fit_prefill(model_cfg, chunks, shares, times_ms):
    """Grid over (r_sat, lambda); closed-form C per grid point (log-LSQ)."""
    ops = nx.prefill_batch_workloads(model_cfg, chunks)
    flops = sum(o.flops for o in ops)
    best = None
    for r_sat in [i / 100.0 for i in range(30, 101)]:
        for lam in np.arange(0.0, 1.0001, 0.02):
            f = [1.0 / s if s <= r_sat else (1.0 / r_sat) * (1.0 + lam * (s - r_sat)) for s in shares]
            logc = statistics.mean(math.log(flops * fi) - math.log(t * 1e-3) for fi, t in zip(f, times_ms))
            C = math.exp(logc)
            err = sum((math.log(flops * fi / C) - math.log(t * 1e-3)) ** 2 for fi, t in zip(f, times_ms))
            if best is None or err < best[0]:
                best = (err, float(r_sat), float(lam), C)
    return {"r_sat": best[1], "lambda": best[2], "peak_compute": best[3], "rms_log_err": math.sqrt(best[0] / len(shares))}


def fit_decode(model_cfg, ctx, shares, times_ms):
    ops = nx.decode_op_workloads(model_cfg, ctx)
    mem = sum(o.mem_bytes for o in ops)
    best = None
    for sat in [i / 100.0 for i in range(5, 101)]:
        f = [1.0 if s >= sat else sat / s for s in shares]
        logb = statistics.mean(math.log(mem * fi) - math.log(t * 1e-3) for fi, t in zip(f, times_ms))
        B = math.exp(logb)
        err = sum((math.log(mem * fi / B) - math.log(t * 1e-3)) ** 2 for fi, t in zip(f, times_ms))
        if best is None or err < best[0]:
            best = (err, float(sat), B)
    return {"bw_sat": best[1], "peak_bandwidth": best[2], "rms_log_err": math.sqrt(best[0] / len(shares))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--ref-model", default="8b", help="reference ModelConfig preset for the cost model")
    ap.add_argument("--ref-dims", default=None,
                    help="hidden,ffn,layers,heads,elem_bytes for ModelConfig::derive when the reference has no "
                         "preset (e.g. 8192,28672,80,64,2 for Llama-3.1-70B)")
    ap.add_argument("--out", default="profiles/b200_llama3_8b")
    ap.add_argument("--decode-batch", type=int, default=64)
    ap.add_argument("--decode-ctx", type=int, default=600)
    ap.add_argument("--prefill-chunks", default="512,512,512,512")
    ap.add_argument("--from-json", default=None,
                    help="refit from the sweeps stored in an earlier calibration JSON (no device)")
    args = ap.parse_args()

    if args.from_json:
        old = json.load(open(args.from_json))
        b = old["batches"]
        fit_and_write(args, old["sweep"], old["contention"], old["sm_count"], b["prefill_chunks"],
                      b["decode_batch"], b["decode_ctx"])
        return
    pref = [int(x) for x in args.prefill_chunks.split(",")]
    B, ctx = args.decode_batch, args.decode_ctx
    pages_per = (max(ctx, max(pref)) + 15) // 16 + 1
    dev = D.Device(D.arch_preset(args.model), num_pages=(B + len(pref)) * pages_per + 64,
                   max_decode_batch=max(64, B), max_prefill_tokens=max(2048, sum(pref)) + 128)
    info = dev.info()
    total = info.sm_count
    rng = np.random.default_rng(0)
    vocab = dev.arch.vocab
    nxt = [0]

    def pages(n):
        p = list(range(nxt[0], nxt[0] + n))
        nxt[0] += n
        return p

    P = [dict(tokens=rng.integers(0, vocab, n).tolist(), start=0, pages=pages(pages_per)) for n in pref]
    Dm = [dict(tokens=[int(rng.integers(0, vocab))], start=ctx - 1, pages=pages(pages_per)) for _ in range(B)]
    layouts = [(info.layout_decode_sms[k], info.layout_prefill_sms[k]) for k in range(info.n_layouts)]
    pct = lambda sms: int(round(100.0 * sms / total))  # noqa: E731

    sweep = {"prefill": [], "decode": []}
    for d_sms, p_sms in layouts:
        t, ops = measure(dev, Dm, 1, pct(d_sms))
        sweep["decode"].append({"sms": d_sms, "ms": t, "op_ms": ops})
        t, ops = measure(dev, P, 0, pct(p_sms))
        sweep["prefill"].append({"sms": p_sms, "ms": t, "op_ms": ops})
    t, ops = measure(dev, Dm, 1, 100)
    sweep["decode"].append({"sms": total, "ms": t, "op_ms": ops})
    t, ops = measure(dev, P, 0, 100)
    sweep["prefill"].append({"sms": total, "ms": t, "op_ms": ops})

    # co-location: decode on its partition while a prefill batch runs on the other
    contention = []
    for d_sms, p_sms in layouts:
        if d_sms not in (16, 24, 32, 40, 48, 64, 72, 80, 96, 112):
            continue
        alone = next(x["ms"] for x in sweep["decode"] if x["sms"] == d_sms)
        co = []
        for _ in range(8):
            dev.launch(P, lane=0, sm_pct=pct(p_sms))
            dev.launch(Dm, lane=1, sm_pct=pct(d_sms))
            co.append(dev.wait(1)[1])
            dev.wait(0)
        contention.append({"decode_sms": d_sms, "prefill_sms": p_sms, "decode_alone_ms": alone,
                           "decode_colocated_ms": statistics.median(co),
                           "slowdown": statistics.median(co) / alone})

    fit_and_write(args, sweep, contention, total, pref, B, ctx)


def fit_and_write(args, sweep, contention, total, pref, B, ctx):
    m = nx.derive(*[int(v) for v in args.ref_dims.split(",")]) if args.ref_dims else nx.model_preset(args.ref_model)
    pshares = [x["sms"] / total for x in sweep["prefill"]]
    dshares = [x["sms"] / total for x in sweep["decode"]]
    pf = fit_prefill(m, [(n, n) for n in pref], pshares, [x["ms"] for x in sweep["prefill"]])
    df = fit_decode(m, [ctx] * B, dshares, [x["ms"] for x in sweep["decode"]])
    # per-operator curves: the prefill operators' compute curves from their own
    # sweep times (peak_compute fixed to the phase fit), the decode operators'
    # bandwidth shares from theirs (peak_bandwidth fixed)
    pops = nx.prefill_batch_workloads(m, [(n, n) for n in pref])
    dops = nx.decode_op_workloads(m, [ctx] * B)
    pflops, dmem = op_sums(pops, "flops"), op_sums(dops, "mem_bytes")
    prof = nx.lib().nx_kernel_profile_default()
    per_op = {}
    for k in (0, 1, 3, 4):
        c = fit_curve(pflops[k], pshares, [x["op_ms"][k] for x in sweep["prefill"]], pf["peak_compute"])
        per_op[OPS[k]] = c
        cur = getattr(prof, OPS[k])
        cur.r_sat, cur.lambda_ = c["r_sat"], c["lambda"]
    bw_sat = [df["bw_sat"]] * 5
    for k in (0, 2, 3, 4):
        b = fit_bw_sat(dmem[k], dshares, [x["op_ms"][k] for x in sweep["decode"]], df["peak_bandwidth"])
        per_op.setdefault(OPS[k], {})["bw_sat"] = b["bw_sat"]
        per_op[OPS[k]]["bw_rms_log_err_shape"] = b["rms_log_err_shape"]
        bw_sat[k] = b["bw_sat"]
    cf = fit_contention(contention)
    out = {
        "model": args.model, "ref_model_preset": args.ref_model, "ref_dims": args.ref_dims, "sm_count": total,
        "gpu_spec": {"total_sm": total, "peak_compute": pf["peak_compute"], "peak_bandwidth": df["peak_bandwidth"]},
        "profile": {k: {"r_sat": getattr(prof, k).r_sat, "lambda": getattr(prof, k).lambda_} for k in OPS},
        "bw_sat": bw_sat, "contention": contention,
        "contention_fit": cf,
        "fit": {"prefill": pf, "decode": df, "per_op": per_op},
        "sweep": sweep,
        "batches": {"prefill_chunks": pref, "decode_batch": B, "decode_ctx": ctx},
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    with open(args.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    with open(args.out + ".calib", "w") as f:
        f.write("# B200 refit (paper_2507_06608_b200.calibrate): " + args.model + "\n")
        f.write(nx.kernel_profile_text(prof))
    print(json.dumps({k: out[k] for k in ("gpu_spec", "profile", "bw_sat", "contention_fit")}))


if __name__ == "__main__":
    main()

"""On-device profiler -> cost-model calibration.

Measures, on the real B200 partitions, the latency of a representative
prefill batch and decode batch of the served model on every pre-instantiated
green-context layout (the diminishing-returns curves of PAPER.md:462-464),
plus decode latency alone vs co-located with a prefill batch (the contention
the cost model's B_decode term predicts). It then refits the
cost model so its predictions match the device:

  * GpuSpec.peak_compute / peak_bandwidth := effective full-GPU rates;
  * per-operator (r_sat, lambda) of Eq. 5 from the prefill sweep;
  * per-operator bw_sat of the flagged bandwidth extension (nx_cost_ext)
    from the decode sweep.

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


def measure(dev, members, lane, pct, reps=5, warm=2):
    for _ in range(warm):
        dev.forward(members, lane=lane, sm_pct=pct)
    ts = [dev.forward(members, lane=lane, sm_pct=pct)[2] for _ in range(reps)]
    return statistics.median(ts)


def fit_prefill(model_cfg, chunks, shares, times_ms):
    """Grid over (r_sat, lambda); closed-form C per grid point (log-LSQ)."""
    ops = nx.prefill_batch_workloads(model_cfg, chunks)
    flops = sum(o.flops for o in ops)
    best = None
    for r_sat in np.arange(0.30, 1.0001, 0.01):
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
    for sat in np.arange(0.05, 1.0001, 0.01):
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
    args = ap.parse_args()

    pref = [int(x) for x in args.prefill_chunks.split(",")]
    B, ctx = args.decode_batch, args.decode_ctx
    pages_per = (max(ctx, max(pref)) + 15) // 16 + 1
    dev = D.Device(D.arch_preset(args.model), num_pages=(B + len(pref)) * pages_per + 64)
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
        sweep["decode"].append({"sms": d_sms, "ms": measure(dev, Dm, 1, pct(d_sms))})
        sweep["prefill"].append({"sms": p_sms, "ms": measure(dev, P, 0, pct(p_sms))})
    sweep["decode"].append({"sms": total, "ms": measure(dev, Dm, 1, 100)})
    sweep["prefill"].append({"sms": total, "ms": measure(dev, P, 0, 100)})

    # co-location: decode on its partition while a prefill batch runs on the other
    contention = []
    for d_sms, p_sms in layouts:
        if d_sms not in (32, 48, 64, 72, 80, 96, 112):
            continue
        alone = next(x["ms"] for x in sweep["decode"] if x["sms"] == d_sms)
        co = []
        for _ in range(4):
            dev.launch(P, lane=0, sm_pct=pct(p_sms))
            dev.launch(Dm, lane=1, sm_pct=pct(d_sms))
            co.append(dev.wait(1)[1])
            dev.wait(0)
        contention.append({"decode_sms": d_sms, "prefill_sms": p_sms, "decode_alone_ms": alone,
                           "decode_colocated_ms": statistics.median(co),
                           "slowdown": statistics.median(co) / alone})

    m = nx.derive(*[int(v) for v in args.ref_dims.split(",")]) if args.ref_dims else nx.model_preset(args.ref_model)
    pf = fit_prefill(m, [(n, n) for n in pref], [x["sms"] / total for x in sweep["prefill"]],
                     [x["ms"] for x in sweep["prefill"]])
    df = fit_decode(m, [ctx] * B, [x["sms"] / total for x in sweep["decode"]], [x["ms"] for x in sweep["decode"]])
    prof = nx.lib().nx_kernel_profile_default()
    for name in ("qkv_proj", "attn_prefill", "attn_out_proj", "ffn"):
        c = getattr(prof, name)
        c.r_sat, c.lambda_ = pf["r_sat"], pf["lambda"]
    bw_sat = [df["bw_sat"]] * 5
    out = {
        "model": args.model, "ref_model_preset": args.ref_model, "sm_count": total,
        "gpu_spec": {"total_sm": total, "peak_compute": pf["peak_compute"], "peak_bandwidth": df["peak_bandwidth"]},
        "profile": {"r_sat": pf["r_sat"], "lambda": pf["lambda"]}, "bw_sat": bw_sat,
        "fit": {"prefill": pf, "decode": df}, "sweep": sweep, "contention": contention,
        "batches": {"prefill_chunks": pref, "decode_batch": B, "decode_ctx": ctx},
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    with open(args.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    with open(args.out + ".calib", "w") as f:
        f.write("# B200 refit (paper_2507_06608_b200.calibrate): " + args.model + "\n")
        f.write(nx.kernel_profile_text(prof))
    print(json.dumps({k: out[k] for k in ("gpu_spec", "profile", "bw_sat", "fit", "contention")}))


if __name__ == "__main__":
    main()

"""Serving capacity: the highest Poisson arrival rate at which an engine keeps
>= 90% of requests inside both SLOs (TTFT <= --slo-ttft and per-request p99
TBT <= --slo-tbt) -- the paper's "highest arrival rate ... without violating
token latency constraints", measured on the device clock.

For every engine (nexus, static at given shares, monolithic chunked prefill;
same kernels, same device), the rate is bisected; each probe serves
--requests ShareGPT-shaped requests for each of --seeds (held out from the
controller sweeps) and pools the attainment. Writes one JSON line per probe
and a summary JSON.

    python tools/capacity.py --engines nexus,static79,static50,monolithic --lo 64 --hi 192
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2507_06608_b200 as nx  # noqa: E402
from paper_2507_06608_b200 import device as D  # noqa: E402


def bisect_capacity(attainment_at, lo, hi, tol, target):
    """Highest rate in [lo, hi] whose attainment meets `target`, to within
    `tol` (attainment assumed non-increasing in the rate)."""
    if attainment_at(lo) < target:
        return {"capacity_rps": None, "note": f"below target at {lo}"}
    if hi <= lo or attainment_at(hi) >= target:
        return {"capacity_rps": hi, "note": "target met at the upper bound"}
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if attainment_at(mid) >= target:
            lo = mid
        else:
            hi = mid
    return {"capacity_rps": lo, "first_failing_rps": hi}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--workload", default="sharegpt")
    ap.add_argument("--engines", default="nexus,static79,monolithic")
    ap.add_argument("--lo", type=float, default=64.0)
    ap.add_argument("--hi", type=float, default=192.0)
    ap.add_argument("--tol", type=float, default=4.0)
    ap.add_argument("--requests", type=int, default=2000)
    ap.add_argument("--seeds", default="201,202,203")
    ap.add_argument("--target", type=float, default=0.9)
    ap.add_argument("--beta", type=float, default=2.0)
    ap.add_argument("--gamma", type=float, default=5000.0)
    ap.add_argument("--max-decode-batch", type=int, default=128)
    ap.add_argument("--token-budget", type=int, default=2048, help="prefill tokens per batch (both engines)")
    ap.add_argument("--kv-gb", type=float, default=80.0)
    ap.add_argument("--decode-target-ms", type=float, default=0.0, help="nexus decode-step target (bench.py)")
    ap.add_argument("--slo-ttft", type=float, default=1.0)
    ap.add_argument("--slo-tbt", type=float, default=0.05)
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "capacity"))
    args = ap.parse_args()
    calib = os.path.join(REPO, "profiles", "b200_" + args.model.replace(".", "_").replace("-", "_"))
    page = 16
    num_pages = int(args.kv_gb * (1 << 30) // (page * bench.MODELS[args.model][1]))
    dev = D.Device(D.arch_preset(args.model), num_pages=num_pages, page_tokens=page,
                   max_prefill_tokens=args.token_budget + args.max_decode_batch, max_decode_batch=args.max_decode_batch)
    vocab = dev.arch.vocab
    seeds = [int(x) for x in args.seeds.split(",")]
    probes = open(args.out + ".jsonl", "a")

    def engine_cfg(name):
        kind, share = name, 50
        if name.startswith("static"):
            kind, share = "static", int(name[6:] or 50)
        return bench.make_cfg(nx, kind, num_pages, page, nx.NX_CLOCK_DEVICE, calib, True, args.max_decode_batch,
                              1.3, args.beta, args.model, args.gamma, share, 1, args.token_budget,
                              args.decode_target_ms / 1e3 if kind == "nexus" else 0.0)

    def probe(name, rate):
        cfg = engine_cfg(name)
        tot = good = 0
        ttft, tbt = [], []
        t0 = time.time()
        for seed in seeds:
            trace = nx.workload_trace(args.workload, rate, args.requests, seed)
            rng = np.random.default_rng(seed)
            eng = nx.Engine(cfg, device=dev)
            eng.set_logging(True, False)
            for t in trace:
                eng.submit(t, rng.integers(0, vocab, t.prompt_len, dtype=np.int32).tolist())
            eng.run()
            m = bench.log_metrics(eng.event_log(), args.slo_ttft, args.slo_tbt)
            eng.close()
            tot += m["completed"]
            good += m["good_requests"]
            ttft += m["ttft"]
            tbt += m["tbt"]
        att = good / tot if tot else 0.0
        row = {"engine": name, "rate": rate, "attainment": att, "requests": tot,
               "ttft_p50": bench.nearest_rank(ttft, 50), "ttft_p99": bench.nearest_rank(ttft, 99),
               "tbt_p50": bench.nearest_rank(tbt, 50), "tbt_p99": bench.nearest_rank(tbt, 99),
               "wall_s": time.time() - t0}
        probes.write(json.dumps(row) + "\n")
        probes.flush()
        print(json.dumps(row), flush=True)
        return att

    summary = {}
    for name in args.engines.split(","):
        summary[name] = bisect_capacity(lambda rate: probe(name, rate), args.lo, args.hi, args.tol, args.target)
    summary["config"] = {"model": args.model, "workload": args.workload, "requests_per_seed": args.requests,
                         "seeds": seeds, "target_attainment": args.target,
                         "slo": {"ttft_s": args.slo_ttft, "tbt_p99_s": args.slo_tbt}, "beta": args.beta,
                         "gamma": args.gamma, "max_decode_batch": args.max_decode_batch,
                         "token_budget": args.token_budget}
    json.dump(summary, open(args.out + ".json", "w"), indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()

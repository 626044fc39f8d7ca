"""C5: arrival-rate sweep of Nexus vs a fixed 50/50 split vs non-partitioned
chunked prefill, same kernels, same trace per rate.

One device (weights, KV cache, green-context layouts) is loaded once; every
(engine, rate) point serves the identical trace on a fresh engine with the
device clock. Writes one JSON line per point and a markdown table.

    python tools/rate_sweep.py --rates 32,64,96,128 --requests 400 --out profiles/r01_rate_sweep_8b
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2507_06608_b200 as nx  # noqa: E402
from paper_2507_06608_b200 import device as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--workload", default="sharegpt")
    ap.add_argument("--rates", default="32,64,96,128")
    ap.add_argument("--requests", type=int, default=400)
    ap.add_argument("--engines", default="nexus,static,monolithic")
    ap.add_argument("--beta", type=float, default=2.0)
    ap.add_argument("--gamma", type=float, default=5000.0, help="SPF aging (bench.py default)")
    ap.add_argument("--max-decode-batch", type=int, default=128)
    ap.add_argument("--kv-gb", type=float, default=80.0)
    ap.add_argument("--slo-ttft", type=float, default=1.0)
    ap.add_argument("--slo-tbt", type=float, default=0.05)
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "r01_rate_sweep_8b"))
    args = ap.parse_args()
    calib = os.path.join(REPO, "profiles", "b200_" + args.model.replace(".", "_").replace("-", "_"))
    page = 16
    num_pages = int(args.kv_gb * (1 << 30) // (page * bench.MODELS[args.model][1]))
    dev = D.Device(D.arch_preset(args.model), num_pages=num_pages, page_tokens=page,
                   max_prefill_tokens=2048 + args.max_decode_batch, max_decode_batch=args.max_decode_batch)
    vocab = dev.arch.vocab
    rows = []

    def serve(engine, rate, seed):
        cfg = bench.make_cfg(nx, engine, num_pages, page, nx.NX_CLOCK_DEVICE, calib, True,
                             args.max_decode_batch, 1.3, args.beta, args.model, args.gamma)
        trace = nx.workload_trace(args.workload, rate, args.requests, seed)
        rng = np.random.default_rng(seed)
        eng = nx.Engine(cfg, device=dev)
        eng.set_logging(True, False)
        for t in trace:
            eng.submit(t, rng.integers(0, vocab, t.prompt_len, dtype=np.int32).tolist())
        eng.run()
        m = bench.log_metrics(eng.event_log(), args.slo_ttft, args.slo_tbt)
        st = eng.stats()
        eng.close()
        return m, st

    serve("nexus", float(args.rates.split(",")[0]), 999)  # warm-up
    for rate in [float(r) for r in args.rates.split(",")]:
        for engine in args.engines.split(","):
            m, st = serve(engine, rate, 7 + int(rate))
            row = {"engine": engine, "rate": rate, "goodput": m["good_tokens"] / m["window"],
                   "slo_attainment": m["good_tokens"] / m["out_tokens"],
                   "ttft_p50": bench.nearest_rank(m["ttft"], 50), "ttft_p99": bench.nearest_rank(m["ttft"], 99),
                   "tbt_p50": bench.nearest_rank(m["tbt"], 50), "tbt_p99": bench.nearest_rank(m["tbt"], 99),
                   "switches": st.switches, "completed": m["completed"]}
            rows.append(row)
            print(json.dumps(row), flush=True)
    with open(args.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    lines = [f"# Rate sweep: {args.model}, {args.workload}, {args.requests} requests per point, "
             f"SLO TTFT <= {args.slo_ttft}s & p99 TBT <= {1000 * args.slo_tbt:.0f} ms, beta {args.beta}, gamma {args.gamma:g}, "
             f"max decode batch {args.max_decode_batch}", "",
             "| rate | engine | goodput tok/s | SLO attain | TTFT p50/p99 ms | TBT p50/p99 ms |",
             "|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['rate']:.0f} | {r['engine']} | {r['goodput']:.0f} | {r['slo_attainment']:.3f} | "
                     f"{1e3 * r['ttft_p50']:.0f} / {1e3 * r['ttft_p99']:.0f} | "
                     f"{1e3 * r['tbt_p50']:.1f} / {1e3 * r['tbt_p99']:.1f} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()

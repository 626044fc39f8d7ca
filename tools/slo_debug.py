"""Per-request SLO breakdown of one device-clock run (which requests miss the
TTFT or the per-request p99 TBT SLO, and by how much)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2507_06608_b200 as nx  # noqa: E402
from paper_2507_06608_b200 import device as D  # noqa: E402

ENGINE = os.environ.get("ENGINE", "nexus")
RATE = float(os.environ.get("RATE", "96"))
N = int(os.environ.get("N", "2000"))
MDB = int(os.environ.get("MDB", "128"))
BETA = float(os.environ.get("BETA", "2.0"))
calib = os.path.join(REPO, "profiles", "b200_llama3_8b")
num_pages = int(80.0 * (1 << 30) // (16 * bench.MODELS["llama3-8b"][1]))
dev = D.Device(D.arch_preset("llama3-8b"), num_pages=num_pages, max_prefill_tokens=2048 + MDB, max_decode_batch=MDB)
cfg = bench.make_cfg(nx, ENGINE, num_pages, 16, nx.NX_CLOCK_DEVICE, calib, True, MDB, 1.3, BETA, "llama3-8b", 5000.0)
trace = nx.workload_trace("sharegpt", RATE, N, 201)
rng = np.random.default_rng(201)
eng = nx.Engine(cfg, device=dev)
for t in trace:
    eng.submit(t, rng.integers(0, dev.arch.vocab, t.prompt_len, dtype=np.int32).tolist())
eng.run()
arrival, times = {}, {}
for line in eng.event_log().splitlines():
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
miss_ttft = miss_tbt = 0
hist = {}
for rid, ts in times.items():
    tt = ts[0] - arrival[rid]
    gaps = sorted(b - a for a, b in zip(ts, ts[1:]))
    p99 = gaps[max(0, -(-99 * len(gaps) // 100) - 1)] if gaps else 0.0
    if tt > 1.0:
        miss_ttft += 1
    if p99 > 0.05:
        miss_tbt += 1
        k = min(len(ts), 400) // 50 * 50
        hist[k] = hist.get(k, 0) + 1
        if miss_tbt <= 8:
            big = [round(g * 1e3, 1) for g in gaps[-5:]]
            print("miss", rid, "tokens", len(ts), "ttft", round(tt, 3), "largest gaps ms", big)
print("requests", len(times), "miss_ttft", miss_ttft, "miss_tbt", miss_tbt, "miss by output length bucket", sorted(hist.items()))
# decode launches: batch size, applied share, latency
dl = []
for line in eng.event_log().splitlines():
    c = line.split("\t")
    if c[2] == "launch" and c[1] == "decode":
        dl.append((len(c[3].split(",")), int(c[4]), float(c[6])))
if dl:
    big = sorted(dl, key=lambda x: -x[2])[:5]
    print("decode launches", len(dl), "mean rows", round(sum(x[0] for x in dl) / len(dl), 1),
          "mean ms", round(1e3 * sum(x[2] for x in dl) / len(dl), 2), "slowest (rows, r_p, ms)",
          [(a, b, round(1e3 * c, 1)) for a, b, c in big])

# prefill-lane composition: tokens per prefill (or mixed) batch, its latency, lane busy time
sizes, lats, dec_rows, busy = [], [], [], 0.0
for line in eng.event_log().splitlines():
    c = line.split("\t")
    if c[2] != "launch" or c[1] not in ("prefill", "mixed"):
        continue
    pre = d = 0
    for m in c[3].split(","):
        rid, tok, _ = (int(x) for x in m.split(":"))
        if c[1] == "prefill" or tok > 1:
            pre += tok
        else:
            d += 1
    sizes.append(pre)
    dec_rows.append(d)
    lats.append(float(c[6]) if len(c) > 6 else 0.0)
sizes_s = sorted(sizes)
print("prefill-lane batches", len(sizes), "mean prefill tokens", round(sum(sizes) / len(sizes)), "p50", sizes_s[len(sizes) // 2],
      "mean decode rows", round(sum(dec_rows) / len(dec_rows), 1), "mean latency ms", round(1e3 * sum(lats) / len(lats), 2),
      "busy s", round(sum(lats), 2))

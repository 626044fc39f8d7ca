"""One-line digest of bench.py JSON lines: this engine vs the same-trace baselines."""
import json
import sys


def brief(path):
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "value" not in d:
            continue
        c = d.get("config", {})
        out = [f"{path}: beta {c.get('beta')} budget {c.get('token_budget')} mdb {c.get('max_decode_batch')}",
               f"  nexus      goodput {d['value']:.0f}  ttft p50/p99 {d['ttft_p50']:.3f}/{d['ttft_p99']:.3f}"
               f"  tbt p50/p99 {1e3 * d['tbt_p50']:.1f}/{1e3 * d['tbt_p99']:.1f} ms  att {d['slo_attainment']:.3f}"
               f"  r_p {d.get('r_p_hist_arrivals')}"]
        for name, b in d.get("same_kernel_baselines", {}).items():
            m = b["this_engine_same_traces"]
            out.append(f"  same traces: nexus {m['goodput']:.0f} {m['ttft_p99']:.3f} s {1e3 * m['tbt_p99']:.1f} ms"
                       f" | {name} {b['goodput']:.0f} {b['ttft_p99']:.3f} s {1e3 * b['tbt_p99']:.1f} ms")
        print("\n".join(out))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        brief(p)

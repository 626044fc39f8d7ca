"""Contention refit report: the cost model's co-located decode
slowdown (decode_latency_contended / phase_latency_isolated, costmodel.cpp:56-96,
with the refit GpuSpec, profile and bw_sat of a calibration) against the slowdown
measured on the B200 partitions by paper_2507_06608_b200.calibrate.

    python tools/contention_report.py profiles/b200_llama3_8b > profiles/r01s2_contention_refit.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_06608_b200 as nx  # noqa: E402


def main(base):
    cal = json.load(open(base + ".json"))
    m = (nx.derive(*[int(v) for v in cal["ref_dims"].split(",")]) if cal.get("ref_dims")
         else nx.model_preset(cal["ref_model_preset"]))
    gs = cal["gpu_spec"]
    gpu = nx.gpu_spec(gs["total_sm"], gs["peak_compute"], gs["peak_bandwidth"], 150 << 30)
    prof, _ = nx.parse_kernel_profile(open(base + ".calib").read())
    nx.set_cost_ext(cal["bw_sat"])
    try:
        report(cal, m, gpu, prof)
    finally:
        nx.set_cost_ext(None)  # process-wide switch: leave the reference form on
    cf = cal.get("contention_fit")
    if cf:
        report_fit(cal, cf)


def report_fit(cal, cf):
    c2 = cf.get("c2", 0.0)
    print("\nFitted measured-contention term (nx_cost_ext.contention, flagged): slowdown = "
          f"{cf['c0']:.4f} + {cf['c1']:.4f} p + {c2:.4f} p^2, p = prefill share\n")
    print("| decode SMs | prefill share | measured slowdown | fitted slowdown | rel. error |")
    print("|---|---|---|---|---|")
    for c in cal["contention"]:
        p = c["prefill_sms"] / (c["prefill_sms"] + c["decode_sms"])
        f = cf["c0"] + cf["c1"] * p + c2 * p * p
        print(f"| {c['decode_sms']} | {p:.3f} | {c['slowdown']:.3f} | {f:.3f} | {f / c['slowdown'] - 1:+.3f} |")


def report(cal, m, gpu, prof):
    b = cal["batches"]
    dops = nx.decode_op_workloads(m, [b["decode_ctx"]] * b["decode_batch"])
    pops = nx.prefill_batch_workloads(m, [(n, n) for n in b["prefill_chunks"]])
    total = cal["sm_count"]
    print(f"# Contention refit report: {cal['model']} (profiles/b200_{cal['model'].replace('.', '_').replace('-', '_')}.json)\n")
    print("Decode batch B = %d x ctx %d beside a prefill batch of %s tokens; model = the reference"
          % (b["decode_batch"], b["decode_ctx"], "+".join(map(str, b["prefill_chunks"]))))
    print("contended-decode formula (B_decode, costmodel.cpp:56-96) on the refit spec with the")
    print("bandwidth-share extension (bw_sat = %.2f).\n" % cal["bw_sat"][0])
    print("| decode SMs | prefill SMs | measured alone ms | measured co-located ms | measured slowdown | model alone ms | model co-located ms | model slowdown |")
    print("|---|---|---|---|---|---|---|---|")
    for c in cal["contention"]:
        sd, sp = c["decode_sms"] / total, c["prefill_sms"] / total
        alone = nx.phase_latency_isolated(dops, sd, gpu, prof).total_s
        pbd = nx.phase_latency_isolated(pops, sp, gpu, prof)
        co = nx.decode_latency_contended(dops, sd, pbd, pops, gpu, prof).total_s
        print(f"| {c['decode_sms']} | {c['prefill_sms']} | {c['decode_alone_ms']:.2f} | {c['decode_colocated_ms']:.2f} | "
              f"{c['slowdown']:.3f} | {1e3 * alone:.2f} | {1e3 * co:.2f} | {co / alone:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/b200_llama3_8b")

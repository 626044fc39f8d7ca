#!/bin/bash
# 8 warp pairs x 1 stage decode attention: GPU suite, smoke, bench (both engines), C3
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for e in nexus monolithic; do timeout 900 python bench.py --engine $e > gpurun_out/bj_bench_$e.json 2> gpurun_out/bj_bench_$e.err; echo "rc $?"; python -c "
import json; d=json.load(open('gpurun_out/bj_bench_$e.json')); print('$e', round(d['value']), d['ttft_p50'], d['ttft_p99'], d['tbt_p99'], d['slo_attainment'], d['roofline']['frac'], d['roofline']['partition']['frac'], d['e2e']['value'])"; done
timeout 1500 python bench.py --model qwen2.5-14b --workload longbench --rate 2.5 --requests 60 --steps 1 --warmup 1 --engine nexus --slo-ttft 4.0 --slo-tbt 0.075 --max-decode-batch 64 > gpurun_out/bj_c3_nexus.json 2> gpurun_out/bj_c3_nexus.err; python -c "
import json; d=json.load(open('gpurun_out/bj_c3_nexus.json')); print('c3', round(d['value'],1), d['ttft_p50'], d['ttft_p99'], d['tbt_p50'], d['tbt_p99'], d['slo_attainment'])"

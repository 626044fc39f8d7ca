#!/bin/bash
# 8B recalibration on the 8-pair decode attention, then the default bench twice
mkdir -p gpurun_out/bk
timeout 900 python -m paper_2507_06608_b200.calibrate --out gpurun_out/bk/b200_llama3_8b > gpurun_out/bk_calib.log 2>&1; echo "calib rc $?"
cat gpurun_out/bk/b200_llama3_8b.calib
for i in 1 2; do timeout 900 python bench.py --calib gpurun_out/bk/b200_llama3_8b > gpurun_out/bk_bench_$i.json 2> gpurun_out/bk_bench_$i.err; echo "rc $?"; python -c "
import json; d=json.load(open('gpurun_out/bk_bench_$i.json')); print('new-calib', round(d['value']), d['ttft_p50'], d['ttft_p99'], d['tbt_p99'], d['slo_attainment'], d['r_p_hist_arrivals'])"; done

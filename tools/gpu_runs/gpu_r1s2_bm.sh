#!/bin/bash
# decode slack beta on the 8-pair decode attention build
mkdir -p gpurun_out
for beta in 2.25 2.5; do timeout 900 python bench.py --beta $beta > gpurun_out/bm_beta$beta.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bm_beta$beta.json')); print('beta $beta', round(d['value']), d['ttft_p50'], d['ttft_p99'], d['tbt_p99'], d['slo_attainment'], d['r_p_hist_arrivals'])"; done

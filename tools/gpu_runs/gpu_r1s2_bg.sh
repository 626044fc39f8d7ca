mkdir -p gpurun_out
for beta in 1.75 2.25; do timeout 900 python bench.py --beta $beta > gpurun_out/bg_beta$beta.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bg_beta$beta.json').read().strip().splitlines()[-1]); print('beta $beta', round(d['value']), round(d['ttft_p50'],3), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d.get('r_p_hist_arrivals'))"; done

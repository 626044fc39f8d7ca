mkdir -p gpurun_out
for cfg in "2 5000" "2 1000000" "2.5 1500" "2.5 5000"; do set -- $cfg; timeout 900 python bench.py --beta $1 --gamma $2 > gpurun_out/an_b$1_g$2.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/an_b$1_g$2.json').read().strip().splitlines()[-1]); print('beta $1 gamma $2', round(d['value']), round(d['ttft_p50'],3), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d.get('r_p_hist_arrivals'))"; done

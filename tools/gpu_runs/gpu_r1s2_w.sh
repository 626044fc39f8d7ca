mkdir -p gpurun_out
timeout 900 python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b > gpurun_out/w_calib.log 2>&1
cp profiles/b200_llama3_8b.calib profiles/b200_llama3_8b.json gpurun_out/
for beta in 2 2.5 3; do timeout 900 python bench.py --beta $beta > gpurun_out/w_beta$beta.json 2>/dev/null; done
timeout 900 python bench.py --engine monolithic > gpurun_out/w_mono.json 2>/dev/null
for f in gpurun_out/w_beta*.json gpurun_out/w_mono.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d.get('r_p_hist_arrivals'))"; done

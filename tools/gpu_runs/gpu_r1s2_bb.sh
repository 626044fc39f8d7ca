mkdir -p gpurun_out
timeout 1500 python -m paper_2507_06608_b200.calibrate --model llama3-70b --ref-model 70b --ref-dims 8192,28672,80,64,2 --out profiles/b200_llama3_70b > gpurun_out/bb_calib70.log 2>&1; echo "calib rc $?"
tail -c 600 gpurun_out/bb_calib70.log
cp profiles/b200_llama3_70b.calib profiles/b200_llama3_70b.json gpurun_out/ 2>/dev/null
for e in nexus monolithic; do timeout 1200 python bench.py --model llama3-70b --kv-gb 28 --rate 6 --requests 96 --steps 1 --warmup 1 --slo-ttft 2.0 --slo-tbt 0.1 --engine $e > gpurun_out/bb_70b_$e.json 2> gpurun_out/bb_70b_$e.err; echo "rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/bb_70b_$e.json').read().strip().splitlines()[-1]); print('70b $e', round(d['value'],1), round(d['ttft_p50'],2), round(d['ttft_p99'],2), round(d['tbt_p50'],4), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d.get('r_p_hist_arrivals'), d['roofline']['kernel_class'], round(d['roofline']['frac'],3))"; done

mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
for e in nexus monolithic; do timeout 1200 python bench.py --model llama3-70b --kv-gb 28 --rate 6 --requests 96 --steps 1 --warmup 1 --slo-ttft 2.0 --slo-tbt 0.1 --calib none --engine $e > gpurun_out/ba_70b_$e.json 2> gpurun_out/ba_70b_$e.err; echo "rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/ba_70b_$e.json').read().strip().splitlines()[-1]); print('70b $e', round(d['value'],1), round(d['ttft_p50'],2), round(d['ttft_p99'],2), round(d['tbt_p50'],4), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d.get('r_p_hist_arrivals'), d['roofline']['kernel_class'], round(d['roofline']['frac'],3))"; tail -2 gpurun_out/ba_70b_$e.err; done

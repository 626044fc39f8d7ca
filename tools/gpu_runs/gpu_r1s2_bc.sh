mkdir -p gpurun_out
for e in nexus monolithic; do timeout 1200 python bench.py --model llama3-70b --workload bursty --kv-gb 28 --rate 2 --requests 96 --steps 1 --warmup 1 --slo-ttft 2.0 --slo-tbt 0.1 --engine $e > gpurun_out/bd_70b_bursty_$e.json 2> gpurun_out/bd_70b_bursty_$e.err; echo "rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/bd_70b_bursty_$e.json').read().strip().splitlines()[-1]); print('70b bursty $e', round(d['value'],1), round(d['ttft_p50'],2), round(d['ttft_p99'],2), round(d['tbt_p50'],4), round(d['tbt_p99'],4), round(d['slo_attainment'],3))"; done

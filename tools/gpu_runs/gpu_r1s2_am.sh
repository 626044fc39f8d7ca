mkdir -p gpurun_out
for g in 150 500 1500; do timeout 900 python bench.py --gamma $g > gpurun_out/am_gamma$g.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/am_gamma$g.json').read().strip().splitlines()[-1]); print('gamma $g', round(d['value']), round(d['ttft_p50'],3), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3))"; done
timeout 1800 python tools/rate_sweep.py --rates 64,96,112,128,144 --requests 480 --engines nexus,monolithic --out gpurun_out/am_rate_sweep > gpurun_out/am_rate.log 2>&1
cat gpurun_out/am_rate_sweep.md
for e in nexus monolithic; do timeout 1500 python bench.py --model qwen2.5-14b --workload longbench --rate 2.5 --requests 60 --steps 1 --warmup 1 --engine $e --slo-ttft 4.0 --slo-tbt 0.075 --max-decode-batch 64 > gpurun_out/am_c3_$e.json 2> gpurun_out/am_c3_$e.err; python -c "
import json; d=json.loads(open('gpurun_out/am_c3_$e.json').read().strip().splitlines()[-1]); print('c3 $e', round(d['value'],1), round(d['ttft_p50'],2), round(d['ttft_p99'],2), round(d['tbt_p50'],4), round(d['tbt_p99'],4), round(d['slo_attainment'],3))"; done

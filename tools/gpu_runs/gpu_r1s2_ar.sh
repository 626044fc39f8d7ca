mkdir -p gpurun_out
timeout 1800 python tools/rate_sweep.py --rates 64,96,112,128,144,160 --requests 480 --engines nexus,monolithic --out gpurun_out/ar_rate_sweep > gpurun_out/ar_rate.log 2>&1
cat gpurun_out/ar_rate_sweep.md
for e in nexus monolithic; do timeout 1500 python bench.py --model qwen2.5-14b --workload longbench --rate 2.5 --requests 60 --steps 1 --warmup 1 --engine $e --slo-ttft 4.0 --slo-tbt 0.075 --max-decode-batch 64 > gpurun_out/ar_c3_$e.json 2> gpurun_out/ar_c3_$e.err; python -c "
import json; d=json.loads(open('gpurun_out/ar_c3_$e.json').read().strip().splitlines()[-1]); print('c3 $e', round(d['value'],1), round(d['ttft_p50'],2), round(d['ttft_p99'],2), round(d['tbt_p50'],4), round(d['tbt_p99'],4), round(d['slo_attainment'],3))"; done
MODE=prefill REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc2" -s 4 -c 4 -o gpurun_out/ar_prefill_pair python tools/step_driver.py > gpurun_out/ar_ncu.log 2>&1

mkdir -p gpurun_out
timeout 1200 python -m paper_2507_06608_b200.calibrate --model qwen2.5-14b --ref-model 14b --out profiles/b200_qwen2_5_14b > gpurun_out/bf_calib14.log 2>&1; echo "calib rc $?"
cp profiles/b200_qwen2_5_14b.calib profiles/b200_qwen2_5_14b.json gpurun_out/
for e in nexus monolithic; do timeout 1500 python bench.py --model qwen2.5-14b --workload longbench --rate 2.5 --requests 60 --steps 1 --warmup 1 --engine $e --slo-ttft 4.0 --slo-tbt 0.075 --max-decode-batch 64 > gpurun_out/bf_c3_$e.json 2> gpurun_out/bf_c3_$e.err; python -c "
import json; d=json.loads(open('gpurun_out/bf_c3_$e.json').read().strip().splitlines()[-1]); print('c3 $e', round(d['value'],1), round(d['ttft_p50'],2), round(d['ttft_p99'],2), round(d['tbt_p50'],4), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d['config']['gamma'])"; done

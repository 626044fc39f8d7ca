mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/x_pytest.log
tail -3 gpurun_out/x_pytest.log
grep -q "pytest rc 0" gpurun_out/x_pytest.log || exit 1
for b in 64 128; do for dp in 100 33; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done
for p in 100 76; do echo -n "prefill pct=$p "; PPCT=$p MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done
timeout 1200 python -m paper_2507_06608_b200.calibrate --model qwen2.5-14b --ref-model 14b --out profiles/b200_qwen2_5_14b > gpurun_out/x_calib14.log 2>&1
cp profiles/b200_qwen2_5_14b.calib profiles/b200_qwen2_5_14b.json gpurun_out/
for e in nexus monolithic; do timeout 1500 python bench.py --model qwen2.5-14b --workload longbench --rate 2.5 --requests 60 --steps 1 --warmup 1 --engine $e --slo-ttft 4.0 --slo-tbt 0.075 --max-decode-batch 64 > gpurun_out/x_c3_$e.json 2> gpurun_out/x_c3_$e.err; done
for e in nexus monolithic; do python -c "
import json; d=json.loads(open('gpurun_out/x_c3_$e.json').read().strip().splitlines()[-1]); print('$e', round(d['value'],1), round(d['ttft_p50'],2), round(d['ttft_p99'],2), round(d['tbt_p50'],4), round(d['tbt_p99'],4), round(d['slo_attainment'],3))"; done

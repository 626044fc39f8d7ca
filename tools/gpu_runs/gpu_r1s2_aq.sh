mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q > gpurun_out/aq_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/aq_pytest.log
tail -2 gpurun_out/aq_pytest.log
for p in 100 79; do echo -n "prefill pct=$p "; PPCT=$p MODE=prefill REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done > gpurun_out/aq_steps.txt
echo -n "colo 79/21 " >> gpurun_out/aq_steps.txt; B=96 PPCT=79 DPCT=21 DSTEPS=3 MODE=colo REPS=3 timeout 120 python tools/step_driver.py 2>&1 | tail -1 >> gpurun_out/aq_steps.txt
echo -n "decode alone 21% " >> gpurun_out/aq_steps.txt; B=96 DPCT=21 MODE=decode REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1 >> gpurun_out/aq_steps.txt
cat gpurun_out/aq_steps.txt
timeout 900 python bench.py > gpurun_out/aq_bench_nexus.json 2> gpurun_out/aq_bench_nexus.err
python -c "
import json; d=json.loads(open('gpurun_out/aq_bench_nexus.json').read().strip().splitlines()[-1]); print('nexus', round(d['value']), round(d['ttft_p50'],3), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d['roofline'].get('partition'))"

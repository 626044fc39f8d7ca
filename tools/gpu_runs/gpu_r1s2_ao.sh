mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ao_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ao_pytest.log
tail -2 gpurun_out/ao_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/ao_bench_nexus.json 2> gpurun_out/ao_bench_nexus.err
timeout 900 python bench.py --engine monolithic > gpurun_out/ao_bench_mono.json 2> gpurun_out/ao_bench_mono.err
timeout 600 python bench.py --impl reference > gpurun_out/ao_bench_ref.json 2> gpurun_out/ao_bench_ref.err
for f in gpurun_out/ao_bench_nexus.json gpurun_out/ao_bench_mono.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ttft_p50'],3), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d['roofline']['kernel_class'], round(d['roofline']['frac'],3), d['roofline'].get('partition'))"; done
tail -c 400 gpurun_out/ao_bench_ref.json
MODE=prefill PPCT=79 REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ao_launch_prefill79.csv python tools/step_driver.py > /dev/null 2>&1
MODE=prefill REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc2|prefill_attn" -s 4 -c 5 -o gpurun_out/ao_prefill_pair python tools/step_driver.py > gpurun_out/ao_ncu.log 2>&1

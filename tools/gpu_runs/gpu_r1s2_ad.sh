mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ad_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ad_pytest.log
tail -3 gpurun_out/ad_pytest.log
grep -q "pytest rc 0" gpurun_out/ad_pytest.log || exit 1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b > gpurun_out/ad_calib.log 2>&1
cp profiles/b200_llama3_8b.calib profiles/b200_llama3_8b.json gpurun_out/
timeout 900 python bench.py > gpurun_out/ad_bench_nexus.json 2> gpurun_out/ad_bench_nexus.err
timeout 900 python bench.py --engine monolithic > gpurun_out/ad_bench_mono.json 2> gpurun_out/ad_bench_mono.err
for f in gpurun_out/ad_bench_nexus.json gpurun_out/ad_bench_mono.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ttft_p50'],3), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d['roofline']['kernel_class'], round(d['roofline']['frac'],3), d.get('r_p_hist_arrivals'))"; done

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ax_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ax_pytest.log
tail -2 gpurun_out/ax_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/ax_bench_nexus.json 2> gpurun_out/ax_bench_nexus.err
python -c "
import json; d=json.loads(open('gpurun_out/ax_bench_nexus.json').read().strip().splitlines()[-1]); print('nexus', round(d['value']), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), round(d['roofline']['frac'],3), round(d['roofline']['partition']['frac'],3))"

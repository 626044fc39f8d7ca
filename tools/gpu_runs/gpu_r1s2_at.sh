mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/at_bench_nexus.json 2> gpurun_out/at_bench_nexus.err
timeout 900 python bench.py --engine monolithic > gpurun_out/at_bench_mono.json 2> gpurun_out/at_bench_mono.err
timeout 600 python bench.py --impl reference > gpurun_out/at_bench_ref.json 2> gpurun_out/at_bench_ref.err
for f in gpurun_out/at_bench_nexus.json gpurun_out/at_bench_mono.json gpurun_out/at_bench_ref.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ttft_p50'],3), round(d['ttft_p99'],3), round(d['tbt_p99'],4), d.get('slo_attainment'), (d.get('roofline') or {}).get('frac'), d['e2e']['value'])"; done

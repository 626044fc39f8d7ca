mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/z_bench_nexus.json 2> gpurun_out/z_bench_nexus.err
timeout 900 python bench.py --engine monolithic > gpurun_out/z_bench_mono.json 2> gpurun_out/z_bench_mono.err
timeout 600 python bench.py --impl reference > gpurun_out/z_bench_ref.json 2> gpurun_out/z_bench_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/z_smoke.log
for f in gpurun_out/z_bench_nexus.json gpurun_out/z_bench_mono.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ttft_p99'],3), round(d['tbt_p99'],4), round(d['slo_attainment'],3), d['roofline']['kernel_class'], round(d['roofline']['frac'],3), d['e2e']['value'])"; done
tail -2 gpurun_out/z_smoke.log

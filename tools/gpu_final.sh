# End-of-round validation on one B200: GPU test tier, smoke(), default bench line,
# ncu launch list of smoke().
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; tail -3 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -2 gpurun_out/final_smoke.log
timeout 1200 python bench.py --steps 8 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.log; tail -c 300 gpurun_out/final_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; tail -2 gpurun_out/ncu_smoke.log

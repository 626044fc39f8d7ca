mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/a_pytest.log
timeout 900 python bench.py > gpurun_out/a_bench_nexus.json 2> gpurun_out/a_bench_nexus.err
timeout 900 python bench.py --engine monolithic --steps 2 --warmup 3 > gpurun_out/a_bench_mono.json 2> gpurun_out/a_bench_mono.err
tail -3 gpurun_out/a_pytest.log; cat gpurun_out/a_bench_nexus.json gpurun_out/a_bench_mono.json

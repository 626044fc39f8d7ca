set -x
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -30
timeout 600 python bench.py --steps 2 --warmup 1 --requests 60 > gpurun_out/bench_try1.json 2> gpurun_out/bench_try1.err
tail -c 3000 gpurun_out/bench_try1.err
cat gpurun_out/bench_try1.json

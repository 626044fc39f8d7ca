timeout 600 python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b > gpurun_out/calib.json 2> gpurun_out/calib.err
cp profiles/b200_llama3_8b.* gpurun_out/ 2>/dev/null
tail -c 2000 gpurun_out/calib.err
timeout 600 python bench.py --steps 2 --warmup 1 --requests 60 > gpurun_out/bench_try2.json 2> gpurun_out/bench_try2.err
tail -c 2000 gpurun_out/bench_try2.err

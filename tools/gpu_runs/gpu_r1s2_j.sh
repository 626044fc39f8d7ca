mkdir -p gpurun_out
timeout 900 python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b > gpurun_out/j_calib.log 2>&1
tail -3 gpurun_out/j_calib.log
timeout 900 python bench.py > gpurun_out/j_bench_nexus.json 2> gpurun_out/j_bench_nexus.err
timeout 900 python bench.py --engine monolithic --steps 2 > gpurun_out/j_bench_mono.json 2> gpurun_out/j_bench_mono.err
cat gpurun_out/j_bench_nexus.json gpurun_out/j_bench_mono.json

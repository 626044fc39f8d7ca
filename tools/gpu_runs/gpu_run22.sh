timeout 1500 python tools/rate_sweep.py --rates 48,96,128,160 --requests 400 --out gpurun_out/r01_rate_sweep_8b > gpurun_out/sweep8b.log 2>&1
timeout 900 python -m paper_2507_06608_b200.calibrate --model qwen2.5-14b --ref-model 14b --decode-batch 32 --decode-ctx 8192 --prefill-chunks 2048 --out gpurun_out/b200_qwen2_5_14b > gpurun_out/calib14.json 2> gpurun_out/calib14.err
cp gpurun_out/b200_qwen2_5_14b.* profiles/ 2>/dev/null
for eng in nexus monolithic; do
timeout 1200 python bench.py --model qwen2.5-14b --workload longbench --rate 2.5 --requests 60 --steps 1 --warmup 1 --engine $eng --slo-ttft 4.0 --slo-tbt 0.075 --max-decode-batch 64 --kv-gb 100 > gpurun_out/bench14_$eng.json 2> gpurun_out/bench14_$eng.err
done

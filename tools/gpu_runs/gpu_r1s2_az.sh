mkdir -p gpurun_out
timeout 1500 python tools/rate_sweep.py --rates 112,128,144 --requests 480 --engines static --out gpurun_out/az_rate_static > gpurun_out/az_rate.log 2>&1
cat gpurun_out/az_rate_static.md

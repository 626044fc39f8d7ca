timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -5
SMS=16,32,48,64,72,80,96,112,128,148 TOKENS=64 timeout 300 python tools/gemm_sweep.py > gpurun_out/gemm_sweep2.jsonl 2>&1
for eng in nexus monolithic; do for r in 16 32 48 64; do
  timeout 600 python bench.py --engine $eng --rate $r --requests 300 --steps 1 --warmup 1 --profile-every 16 > gpurun_out/sweep_${eng}_${r}.json 2> gpurun_out/sweep_${eng}_${r}.err
done; done

timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
for mdb in 64 128; do for eng in nexus monolithic; do for r in 32 64 96; do
  timeout 600 python bench.py --engine $eng --rate $r --requests 400 --steps 1 --warmup 1 --profile-every 16 --max-decode-batch $mdb > gpurun_out/s2_${eng}_${r}_${mdb}.json 2> gpurun_out/s2_${eng}_${r}_${mdb}.err
done; done; done

timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q 2>&1 | tail -5
SMS=16,32,48,64,72,80,96,112,128,148 TOKENS=64,256 timeout 300 python tools/gemm_sweep.py > gpurun_out/gemm_sweep3.jsonl 2>&1

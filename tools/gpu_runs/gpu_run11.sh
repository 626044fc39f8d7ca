timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe2.jsonl 2>&1

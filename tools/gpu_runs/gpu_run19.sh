timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q 2>&1 | tail -3
timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe5.jsonl 2>&1
SMS=16,32,48,64,96,148 TOKENS=64,128,2048 timeout 300 python tools/gemm_sweep.py > gpurun_out/gemm_sweep5.jsonl 2>&1
MODE=both REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -2
MODE=decode DPCT=22 REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -1

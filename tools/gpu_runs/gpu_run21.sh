timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q 2>&1 | tail -3
SMS=16,24,32,64,148 TOKENS=64 timeout 300 python tools/gemm_sweep.py > gpurun_out/gemm_sweep6.jsonl 2>&1
MODE=both REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -2
MODE=decode DPCT=22 REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -1
MODE=decode DPCT=11 REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -1

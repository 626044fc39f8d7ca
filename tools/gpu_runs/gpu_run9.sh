timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q 2>&1 | tail -5
SMS=16,32,48,64,80,96,112,148 TOKENS=64,2048 timeout 300 python tools/gemm_sweep.py > gpurun_out/gemm_sweep4.jsonl 2>&1
REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -2
REPS=3 DPCT=50 timeout 300 python tools/step_driver.py 2>&1 | tail -1
REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches_decode2.csv python tools/step_driver.py > /dev/null 2>&1

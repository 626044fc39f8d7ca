timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe3.jsonl 2>&1
MODE=both REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -8
MODE=both REPS=4 DPCT=50 PPCT=50 timeout 300 python tools/step_driver.py 2>&1 | tail -4

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q > gpurun_out/aa_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/aa_pytest.log
tail -2 gpurun_out/aa_pytest.log
for p in 100 79; do echo -n "prefill pct=$p "; PPCT=$p MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done
echo -n "decode alone 21% "; B=96 DPCT=21 MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1
echo -n "colo 79/21 "; B=96 PPCT=79 DPCT=21 DSTEPS=3 MODE=colo REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -1
echo -n "colo 79/21 dsteps0 "; B=96 PPCT=79 DPCT=21 DSTEPS=1 MODE=colo REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -1

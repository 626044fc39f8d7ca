mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/d_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/d_pytest.log
for f in 0 1; do for b in 64 128; do for dp in 100 33; do echo -n "fold=$f B=$b DPCT=$dp "; NX_FOLD=$f B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done; done > gpurun_out/d_steps.txt
tail -3 gpurun_out/d_pytest.log; cat gpurun_out/d_steps.txt

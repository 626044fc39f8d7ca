mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/h_pytest.log
for b in 64 128; do for dp in 100 50 33 20; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done > gpurun_out/h_steps.txt
B=64 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/h_launch_dec64.csv python tools/step_driver.py > /dev/null 2>&1
tail -2 gpurun_out/h_pytest.log; cat gpurun_out/h_steps.txt

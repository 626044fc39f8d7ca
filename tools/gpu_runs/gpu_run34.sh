mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
MODE=decode REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -2
MODE=decode REPS=3 DPCT=43 timeout 300 python tools/step_driver.py 2>&1 | tail -2
MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/l34_dec148.csv python tools/step_driver.py > /dev/null 2>&1
MODE=decode REPS=2 DPCT=43 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/l34_dec64.csv python tools/step_driver.py > /dev/null 2>&1

REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -3
REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches_decode.csv python tools/step_driver.py > /dev/null 2>&1
MODE=prefill REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 260 -c 260 --csv --log-file gpurun_out/launches_prefill.csv python tools/step_driver.py > /dev/null 2>&1
ls -la gpurun_out/

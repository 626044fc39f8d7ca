timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_engine.py -x -q 2>&1 | tail -4
MODE=both REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -4
REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches_decode3.csv python tools/step_driver.py > /dev/null 2>&1
MODE=decode REPS=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 3 -c 1 -o gpurun_out/decode_attn2 python tools/step_driver.py > /dev/null 2>&1

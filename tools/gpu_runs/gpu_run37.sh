MODE=prefill REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/l37_pf148.csv python tools/step_driver.py > /dev/null 2>&1
MODE=prefill REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn -s 10 -c 1 -o gpurun_out/pf_attn37 python tools/step_driver.py > /dev/null 2>&1
ls gpurun_out

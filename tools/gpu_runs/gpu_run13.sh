timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe4.jsonl 2>&1
MODE=decode REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -2
MODE=decode REPS=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 3 -c 1 -o gpurun_out/decode_attn python tools/step_driver.py > /dev/null 2>&1

mkdir -p gpurun_out
B=64 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/e_launch_dec64.csv python tools/step_driver.py > /dev/null 2>&1
B=128 DPCT=33 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/e_launch_dec128_33.csv python tools/step_driver.py > /dev/null 2>&1
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 133 -c 4 -o gpurun_out/e_dec64_33_gemm python tools/step_driver.py > gpurun_out/e_ncu_full.log 2>&1
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 1 -o gpurun_out/e_dec64_33_attn python tools/step_driver.py >> gpurun_out/e_ncu_full.log 2>&1
ls -la gpurun_out

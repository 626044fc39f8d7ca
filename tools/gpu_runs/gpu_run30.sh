set -x
mkdir -p gpurun_out
MODE=decode REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -2
MODE=decode REPS=3 DPCT=43 timeout 300 python tools/step_driver.py 2>&1 | tail -2
MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/l30_dec148.csv python tools/step_driver.py > /dev/null 2>&1
MODE=decode REPS=2 DPCT=43 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/l30_dec64.csv python tools/step_driver.py > /dev/null 2>&1
# full captures: qkv (1st gemm of a layer) and o (2nd) of layer 1 in the 2nd decode step at 148 SMs
MODE=decode REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 200 -c 4 -o gpurun_out/g30_dec148 python tools/step_driver.py > /dev/null 2>&1
ls -la gpurun_out

mkdir -p gpurun_out
TOKENS=32,64,128 SMS=16,32,48,64,96,148 timeout 900 python tools/gemm_sweep.py > gpurun_out/b_gemm_sweep.jsonl 2>&1
for dp in 100 50 33; do echo "B=128 DPCT=$dp"; B=128 DPCT=$dp MODE=decode REPS=5 timeout 300 python tools/step_driver.py 2>&1 | tail -2; done > gpurun_out/b_steps.txt
for dp in 100 33; do echo "B=64 DPCT=$dp"; B=64 DPCT=$dp MODE=decode REPS=5 timeout 300 python tools/step_driver.py 2>&1 | tail -2; done >> gpurun_out/b_steps.txt
echo "prefill"; MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -2 >> gpurun_out/b_steps.txt
B=128 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launch_dec128.csv python tools/step_driver.py > /dev/null 2>&1
cat gpurun_out/b_steps.txt

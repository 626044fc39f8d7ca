mkdir -p gpurun_out
T=64 NX_GEMM_DBG=16 timeout 300 python tools/gemm_trace.py > gpurun_out/c_trace64.jsonl 2>&1
for d in 0 1 2 3; do NX_GEMM_DBG=$d T=64 timeout 300 python tools/gemm_dbg.py; done > gpurun_out/c_dbg64.jsonl 2>&1
for d in 0 3; do NX_GEMM_DBG=$d T=128 timeout 300 python tools/gemm_dbg.py; done > gpurun_out/c_dbg128.jsonl 2>&1
for dp in 100 33; do echo "B=128 DPCT=$dp"; B=128 DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done > gpurun_out/c_steps.txt
B=64 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launch_dec64.csv python tools/step_driver.py > /dev/null 2>&1
B=128 DPCT=33 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launch_dec128_33.csv python tools/step_driver.py > /dev/null 2>&1
cat gpurun_out/c_steps.txt

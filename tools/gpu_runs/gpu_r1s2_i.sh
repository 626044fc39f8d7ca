mkdir -p gpurun_out
for mk in 1 8 16 24 32; do for b in 64 128; do for dp in 100 33; do echo -n "minkb=$mk B=$b DPCT=$dp "; NX_DEC_MINKB=$mk B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done; done > gpurun_out/i_steps.txt
cat gpurun_out/i_steps.txt

mkdir -p gpurun_out
T=2048 timeout 300 python tools/gemm_pair_sweep.py > gpurun_out/ac_sweep.jsonl 2>&1; cat gpurun_out/ac_sweep.jsonl
T=1450 SMS=116 timeout 300 python tools/gemm_pair_sweep.py >> gpurun_out/ac_sweep.jsonl 2>&1; tail -4 gpurun_out/ac_sweep.jsonl
for f in 0 1; do for p in 100 79; do echo -n "2cta=$f prefill pct=$p "; NX_GEMM_2CTA=$f PPCT=$p MODE=prefill REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done; done
for f in 0 1; do echo -n "2cta=$f colo 79/21 "; NX_GEMM_2CTA=$f B=96 PPCT=79 DPCT=21 DSTEPS=3 MODE=colo REPS=3 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done

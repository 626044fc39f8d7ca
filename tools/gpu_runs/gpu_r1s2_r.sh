mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r_pytest.log
tail -3 gpurun_out/r_pytest.log
for pl in 512,512,512,512 700,750 655; do for pp in 100 76 52; do for f in 0 1; do echo -n "plens=$pl pct=$pp fit=$f "; NX_BN_FIT=$f PLENS=$pl PPCT=$pp MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done; done > gpurun_out/r_prefill.txt
cat gpurun_out/r_prefill.txt

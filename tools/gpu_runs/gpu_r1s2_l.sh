mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/l_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/l_pytest.log
tail -3 gpurun_out/l_pytest.log
for h in 0 0.85; do echo -n "hybrid=$h "; NX_HYBRID_FRAC=$h MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; echo -n "hybrid=$h pct76 "; NX_HYBRID_FRAC=$h PPCT=76 MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done > gpurun_out/l_prefill.txt
cat gpurun_out/l_prefill.txt
if grep -q "pytest rc 0" gpurun_out/l_pytest.log; then
  for g in 15 1500 5000 1000000; do timeout 900 python bench.py --gamma $g > gpurun_out/l_gamma$g.json 2>/dev/null; done
fi

mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/p_pytest.log
tail -3 gpurun_out/p_pytest.log
for b in 32 64 128; do for dp in 100 33 20; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done
T=64 SMS=32,48,148 timeout 600 python tools/gemm_decode_sweep.py > gpurun_out/p_dec_sweep64.jsonl 2>&1
cat gpurun_out/p_dec_sweep64.jsonl

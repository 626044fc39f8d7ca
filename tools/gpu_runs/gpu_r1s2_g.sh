mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm_decode" > gpurun_out/g_pytest_dec.log 2>&1; echo "rc $?" >> gpurun_out/g_pytest_dec.log
tail -3 gpurun_out/g_pytest_dec.log
T=64 timeout 600 python tools/gemm_decode_sweep.py > gpurun_out/g_dec_sweep64.jsonl 2>&1
T=128 SMS=32,48,148 timeout 600 python tools/gemm_decode_sweep.py > gpurun_out/g_dec_sweep128.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g_pytest.log
for b in 64 128; do for dp in 100 33; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done > gpurun_out/g_steps.txt
cat gpurun_out/g_dec_sweep64.jsonl gpurun_out/g_dec_sweep128.jsonl; tail -3 gpurun_out/g_pytest.log; cat gpurun_out/g_steps.txt

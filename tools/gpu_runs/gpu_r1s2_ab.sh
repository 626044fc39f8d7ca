mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_kernels.py -x -q -k "pair" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ab_pytest.log
tail -30 gpurun_out/ab_pytest.log

set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -40

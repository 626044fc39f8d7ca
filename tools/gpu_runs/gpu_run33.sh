mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q 2>&1 | tail -3
NX_GEMM_DBG=16 timeout 300 python tools/gemm_trace.py
timeout 300 python tools/gemm_dbg.py

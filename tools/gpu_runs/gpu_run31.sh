mkdir -p gpurun_out
for d in 0 1 2 3; do NX_GEMM_DBG=$d timeout 300 python tools/gemm_dbg.py; done > gpurun_out/gemm_dbg.jsonl 2>&1
cat gpurun_out/gemm_dbg.jsonl

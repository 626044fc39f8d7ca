mkdir -p gpurun_out
for d in 3 7 11 15 0 4 8 12; do NX_GEMM_DBG=$d timeout 300 python tools/gemm_dbg.py; done > gpurun_out/gemm_dbg2.jsonl 2>&1
cat gpurun_out/gemm_dbg2.jsonl

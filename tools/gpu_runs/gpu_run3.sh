timeout 300 python tools/gemm_sweep.py > gpurun_out/gemm_sweep.jsonl 2>&1
TOKENS=64 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/gemm_decode python tools/gemm_one.py > gpurun_out/ncu_dec.log 2>&1
TOKENS=2048 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/gemm_prefill python tools/gemm_one.py > gpurun_out/ncu_pre.log 2>&1
tail -3 gpurun_out/ncu_dec.log gpurun_out/ncu_pre.log

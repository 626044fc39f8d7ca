mkdir -p gpurun_out
timeout 120 ./tools/mma_probe 1 > gpurun_out/f_mma1.jsonl 2>&1
timeout 120 ./tools/mma_probe 148 > gpurun_out/f_mma148.jsonl 2>&1
cat gpurun_out/f_mma1.jsonl gpurun_out/f_mma148.jsonl

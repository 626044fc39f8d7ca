set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; tail -3 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -2 gpurun_out/final_smoke.log
timeout 1200 python bench.py --steps 8 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.log; tail -c 300 gpurun_out/final_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 2 -o gpurun_out/decode_attn_short -f env MODEL=llama3-8b B=4 CTX=3000 PCTS=100 REPS=2 python tools/attn_decode_bw.py > gpurun_out/ncu_attn.log 2>&1; tail -3 gpurun_out/ncu_attn.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 2 -o gpurun_out/decode_attn_b128 -f env MODEL=llama3-8b B=128 CTX=1000 PCTS=100 REPS=2 python tools/attn_decode_bw.py > gpurun_out/ncu_attn2.log 2>&1; tail -3 gpurun_out/ncu_attn2.log

mkdir -p gpurun_out
timeout 900 python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b > gpurun_out/q_calib.log 2>&1
cp profiles/b200_llama3_8b.calib profiles/b200_llama3_8b.json gpurun_out/
timeout 900 python bench.py > gpurun_out/q_bench_nexus.json 2> gpurun_out/q_bench_nexus.err
timeout 900 python bench.py --engine monolithic > gpurun_out/q_bench_mono.json 2> gpurun_out/q_bench_mono.err
timeout 600 python bench.py --impl reference > gpurun_out/q_bench_ref.json 2> gpurun_out/q_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/q_launch_bench.csv python bench.py --steps 1 --warmup 0 --requests 120 > /dev/null 2>&1
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_decode -s 133 -c 4 -o gpurun_out/q_dec64_33_gemm python tools/step_driver.py > gpurun_out/q_ncu.log 2>&1
B=64 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_decode -s 133 -c 4 -o gpurun_out/q_dec64_148_gemm python tools/step_driver.py >> gpurun_out/q_ncu.log 2>&1
B=64 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fold_|decode_attn" -s 40 -c 6 -o gpurun_out/q_dec64_148_small python tools/step_driver.py >> gpurun_out/q_ncu.log 2>&1
MODE=prefill REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|prefill_attn" -s 4 -c 5 -o gpurun_out/q_prefill python tools/step_driver.py >> gpurun_out/q_ncu.log 2>&1

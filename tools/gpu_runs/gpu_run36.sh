mkdir -p gpurun_out
timeout 900 python -m paper_2507_06608_b200.calibrate --out gpurun_out/b200_llama3_8b > gpurun_out/calib36.json 2> gpurun_out/calib36.err
tail -3 gpurun_out/calib36.err
timeout 1500 python bench.py --calib gpurun_out/b200_llama3_8b > gpurun_out/bench36.json 2> gpurun_out/bench36.err
tail -c 1500 gpurun_out/bench36.json

timeout 1200 python bench.py > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r01a.json 2> gpurun_out/bench_ref_r01a.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --requests 120 > gpurun_out/bench_ncu.log 2>&1

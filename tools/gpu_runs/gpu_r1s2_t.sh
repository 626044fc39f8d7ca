mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/t_pytest.log
tail -2 gpurun_out/t_pytest.log
timeout 1800 python tools/rate_sweep.py --rates 64,96,112,128,144 --requests 480 --engines nexus,monolithic --out gpurun_out/t_rate_sweep > gpurun_out/t_rate.log 2>&1
cat gpurun_out/t_rate_sweep.md
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 800 --csv --log-file gpurun_out/t_launch_bench.csv python bench.py --steps 1 --warmup 0 --requests 60 > gpurun_out/t_ncu_bench.log 2>&1
tail -5 gpurun_out/t_ncu_bench.log

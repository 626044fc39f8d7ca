mkdir -p gpurun_out
timeout 300 ./tools/bw_probe > gpurun_out/n_bw.jsonl 2>&1
cat gpurun_out/n_bw.jsonl
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q > gpurun_out/n_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/n_pytest.log
tail -2 gpurun_out/n_pytest.log
for p in 100 76; do echo -n "prefill pct=$p "; PPCT=$p MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done
MODE=prefill REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/n_launch_prefill.csv python tools/step_driver.py > /dev/null 2>&1

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ap_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ap_pytest.log
tail -2 gpurun_out/ap_pytest.log
grep -q "pytest rc 0" gpurun_out/ap_pytest.log || exit 1
for w in 0 1; do for p in 100 79; do echo -n "wpol=$w pct=$p "; NX_PAIR_WPOL=$w PPCT=$p MODE=prefill REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done; done
for w in 0 1; do NX_PAIR_WPOL=$w MODE=prefill REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_tc2 -s 4 -c 4 --csv python tools/step_driver.py 2>/dev/null | grep gemm_tc2 | awk -F'","' '{print "wpol='$w'", $(NF-2), $NF}'; done
MODE=prefill PPCT=79 REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ap_launch_prefill79.csv python tools/step_driver.py > /dev/null 2>&1

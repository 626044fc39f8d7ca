mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/y_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/y_pytest.log
tail -3 gpurun_out/y_pytest.log
grep -q "pytest rc 0" gpurun_out/y_pytest.log || exit 1
for b in 64 128; do for dp in 100 33 20; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done
for p in 100 76; do echo -n "prefill pct=$p "; PPCT=$p MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 1 -o gpurun_out/y_dec64_33_attn python tools/step_driver.py > gpurun_out/y_ncu.log 2>&1
B=64 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 1 -o gpurun_out/y_dec64_148_attn python tools/step_driver.py >> gpurun_out/y_ncu.log 2>&1
MODE=prefill REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/y_launch_prefill.csv python tools/step_driver.py > /dev/null 2>&1

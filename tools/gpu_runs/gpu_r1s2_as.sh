mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/as_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/as_pytest.log
tail -2 gpurun_out/as_pytest.log
grep -q "pytest rc 0" gpurun_out/as_pytest.log || exit 1
for b in 64 128; do for dp in 100 33 21; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done; done
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 1 -o gpurun_out/as_dec64_33_attn python tools/step_driver.py > gpurun_out/as_ncu.log 2>&1

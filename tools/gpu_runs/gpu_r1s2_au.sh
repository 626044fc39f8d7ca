mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q > gpurun_out/au_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/au_pytest.log
tail -2 gpurun_out/au_pytest.log
for b in 64 128; do for dp in 33 21; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done; done
B=64 DPCT=33 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_attn -s 33 -c 3 --csv python tools/step_driver.py 2>/dev/null | grep decode_attn | awk -F'","' '{print $NF}'

mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/m_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/m_pytest.log
tail -3 gpurun_out/m_pytest.log
for b in 64 128; do for dp in 100 33 20; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done > gpurun_out/m_steps.txt
cat gpurun_out/m_steps.txt
B=64 DPCT=33 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/m_launch_dec64_33.csv python tools/step_driver.py > /dev/null 2>&1
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 1 -o gpurun_out/m_dec64_33_attn python tools/step_driver.py > gpurun_out/m_ncu.log 2>&1
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_decode -s 133 -c 4 -o gpurun_out/m_dec64_33_gemm python tools/step_driver.py >> gpurun_out/m_ncu.log 2>&1

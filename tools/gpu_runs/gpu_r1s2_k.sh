mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/k_pytest.log
tail -3 gpurun_out/k_pytest.log
for b in 64 128; do for dp in 100 33 20; do echo -n "B=$b DPCT=$dp "; B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done > gpurun_out/k_steps.txt
B=64 DPCT=33 MODE=decode REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/k_launch_dec64_33.csv python tools/step_driver.py > /dev/null 2>&1
B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 1 -o gpurun_out/k_dec64_33_attn python tools/step_driver.py > gpurun_out/k_ncu.log 2>&1
cat gpurun_out/k_steps.txt
if grep -q "pytest rc 0" gpurun_out/k_pytest.log; then
  timeout 900 python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b > gpurun_out/k_calib.log 2>&1
  cp profiles/b200_llama3_8b.calib profiles/b200_llama3_8b.json gpurun_out/
  for beta in 2 3 4 6; do timeout 900 python bench.py --steps 2 --warmup 1 --beta $beta > gpurun_out/k_beta$beta.json 2>/dev/null; done
fi

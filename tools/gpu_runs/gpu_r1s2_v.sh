mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/v_pytest.log
tail -3 gpurun_out/v_pytest.log
for a in pairs pages; do for b in 64 128; do for dp in 100 33; do echo -n "attn=$a B=$b DPCT=$dp "; NX_DEC_ATTN=$a B=$b DPCT=$dp MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done; done; done
for p in 100 76; do echo -n "prefill pct=$p "; PPCT=$p MODE=prefill REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1; done
NX_DEC_ATTN=pairs B=64 DPCT=33 MODE=decode REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 1 -o gpurun_out/v_dec64_33_attn_pairs python tools/step_driver.py > gpurun_out/v_ncu.log 2>&1
MODE=prefill REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_attn -s 1 -c 1 -o gpurun_out/v_prefill_attn python tools/step_driver.py >> gpurun_out/v_ncu.log 2>&1

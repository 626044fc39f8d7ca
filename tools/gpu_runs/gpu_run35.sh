timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pdl in 1 0; do
NX_PDL=$pdl MODE=decode REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -1
NX_PDL=$pdl MODE=decode REPS=3 DPCT=43 timeout 300 python tools/step_driver.py 2>&1 | tail -1
NX_PDL=$pdl MODE=prefill REPS=3 timeout 300 python tools/step_driver.py 2>&1 | tail -1
done

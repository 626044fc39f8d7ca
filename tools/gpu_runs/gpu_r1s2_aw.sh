for pf in 0 4 8 16; do for b in 64 128; do for dp in 33 21; do echo -n "prefetch=$pf B=$b DPCT=$dp "; NX_DEC_PREFETCH=$pf B=$b DPCT=$dp MODE=decode REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done; done; done
for pf in 0 8; do echo -n "prefetch=$pf B=64 full "; NX_DEC_PREFETCH=$pf B=64 DPCT=100 MODE=decode REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done

for r in 1 2; do for v in old new; do
echo -n "$v "; NX_LIB_PATH=ab/$v.so MODE=decode REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1
echo -n "$v "; NX_LIB_PATH=ab/$v.so MODE=decode DPCT=43 REPS=4 timeout 300 python tools/step_driver.py 2>&1 | tail -1
done; done

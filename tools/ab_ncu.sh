for r in 1 2; do for v in old new; do
echo "== $v"; NX_LIB_PATH=ab/$v.so MODE=prefill REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc -s 4 -c 4 --csv python tools/step_driver.py 2>/dev/null | grep gemm | awk -F'","' '{print $NF}'
NX_LIB_PATH=ab/$v.so MODE=decode REPS=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc -s 200 -c 4 --csv python tools/step_driver.py 2>/dev/null | grep gemm | awk -F'","' '{print $NF}'
done; done

for i in 1 2 3 4 5 6; do echo -n "pairpdl run $i "; NX_PAIR_PDL=1 timeout 90 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > /dev/null 2>&1; echo "rc $?"; done
for f in 0 1; do for p in 100 79; do echo -n "pairpdl=$f pct=$p "; NX_PAIR_PDL=$f PPCT=$p MODE=prefill REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done; done

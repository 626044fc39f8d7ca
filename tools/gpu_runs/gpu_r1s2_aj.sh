for i in 1 2 3 4 5; do echo -n "default run $i "; timeout 90 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > /dev/null 2>&1; echo "rc $?"; done
for p in 100 79; do echo -n "prefill pct=$p "; PPCT=$p MODE=prefill REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done

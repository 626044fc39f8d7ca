for i in 1 2 3; do echo -n "pdl0 run $i "; NX_PDL=0 timeout 90 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > /dev/null 2>&1; echo "rc $?"; done
for i in 1 2 3; do echo -n "default run $i "; timeout 90 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > /dev/null 2>&1; echo "rc $?"; done

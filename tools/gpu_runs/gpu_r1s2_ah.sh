mkdir -p gpurun_out
for i in 1 2; do echo "== default run $i"; timeout 100 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > gpurun_out/ah_$i.json 2> gpurun_out/ah_$i.err; echo "rc $?"; done
echo "== green no-fit-single"; NX_HYBRID_FRAC=0 timeout 100 python bench.py --engine monolithic --no-green --steps 1 --warmup 0 --requests 40 > /dev/null 2>&1; echo "rc $?"
echo "== nexus engine"; timeout 150 python bench.py --steps 1 --warmup 0 --requests 40 > gpurun_out/ah_nexus.json 2>&1; echo "rc $?"

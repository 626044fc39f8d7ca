mkdir -p gpurun_out
echo "== fit0"; NX_BN_FIT=0 timeout 120 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > gpurun_out/ag_a.json 2> gpurun_out/ag_a.err; echo "rc $?"; tail -c 200 gpurun_out/ag_a.json
echo "== pdl0"; NX_PDL=0 timeout 120 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > gpurun_out/ag_b.json 2> gpurun_out/ag_b.err; echo "rc $?"; tail -c 200 gpurun_out/ag_b.json
echo "== nogreen"; timeout 120 python bench.py --engine monolithic --no-green --steps 1 --warmup 0 --requests 40 > gpurun_out/ag_c.json 2> gpurun_out/ag_c.err; echo "rc $?"; tail -c 200 gpurun_out/ag_c.json

mkdir -p gpurun_out
for f in 0 1; do echo "== 2cta=$f"; NX_GEMM_2CTA=$f timeout 150 python bench.py --engine monolithic --steps 1 --warmup 0 --requests 40 > gpurun_out/ae_mono$f.json 2> gpurun_out/ae_mono$f.err; echo "rc $?"; tail -c 300 gpurun_out/ae_mono$f.json; tail -3 gpurun_out/ae_mono$f.err; done

for rep in 1 2; do
for c in 0 1; do for f in 0 1; do for p in 100 79; do echo -n "2cta=$c fit=$f pct=$p "; NX_GEMM_2CTA=$c NX_BN_FIT=$f PPCT=$p MODE=prefill REPS=4 timeout 120 python tools/step_driver.py 2>&1 | tail -1; done; done; done
done

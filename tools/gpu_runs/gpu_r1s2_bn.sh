#!/bin/bash
# C5 rate sweep (upper rates) on the 8-pair decode attention build
mkdir -p gpurun_out
timeout 1100 python tools/rate_sweep.py --rates 112,128,144 --requests 480 --engines nexus,monolithic --out gpurun_out/bn_rate_sweep > gpurun_out/bn_rate.log 2>&1; echo "rc $?"
cat gpurun_out/bn_rate_sweep.md

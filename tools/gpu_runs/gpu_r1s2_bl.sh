#!/bin/bash
# ncu --set full of the 8-pair decode attention: C3 shapes on a 32-SM lane (and the 4x3 build for contrast)
mkdir -p gpurun_out
for v in new base; do
  lib=paper_2507_06608_b200/libnexus_b200.so; [ $v = base ] && lib=ab/base.so
  NX_LIB_PATH=$lib MODEL=qwen2.5-14b B=32 CTX=16384 PCTS=21 REPS=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:decode_attn_kernel -s 2 -c 1 -o gpurun_out/ncu_attn_$v -f python tools/attn_decode_bw.py > gpurun_out/ncu_attn_$v.log 2>&1; echo "$v rc $?"
done

#!/bin/bash
# decode-attention bandwidth at C3 and C2 shapes
mkdir -p gpurun_out
MODEL=qwen2.5-14b B=32 CTX=16384 PCTS=100,50,21 OUT=gpurun_out/adbw_c3.jsonl timeout 600 python tools/attn_decode_bw.py 2>&1 | tail -5
MODEL=llama3-8b B=64 CTX=600 PCTS=100,21 OUT=gpurun_out/adbw_8b_64.jsonl timeout 300 python tools/attn_decode_bw.py 2>&1 | tail -3
MODEL=llama3-8b B=128 CTX=4096 PCTS=100,21 OUT=gpurun_out/adbw_8b_128.jsonl timeout 300 python tools/attn_decode_bw.py 2>&1 | tail -3

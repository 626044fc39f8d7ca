#!/bin/bash
# decode attention: warp pairs x ring stages A/B (ab/*.so built with -DNX_DEC_PAIRS/-DNX_DEC_STAGES)
mkdir -p gpurun_out
for v in ${VARS:-base p5s2 p3s4}; do
  echo "== $v"
  NX_LIB_PATH=ab/$v.so timeout 300 python tools/dec_check.py 2>&1 | grep -E "ctx (600|9000) pct (5|30)" | head -4
  for r in 1 2; do
  NX_LIB_PATH=ab/$v.so MODEL=qwen2.5-14b B=32 CTX=16384 PCTS=21,50,100 timeout 300 python tools/attn_decode_bw.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print('$v c3', d['sms'], round(d['attn_us_per_launch'],1), round(d['attn_GBps']), round(d['step_ms'],2))"
  NX_LIB_PATH=ab/$v.so MODEL=llama3-8b B=64 CTX=600 PCTS=21,100 timeout 300 python tools/attn_decode_bw.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print('$v 8b', d['sms'], round(d['attn_us_per_launch'],1), round(d['attn_GBps']), round(d['step_ms'],2))"
  done
done

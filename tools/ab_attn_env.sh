# decode-attention probe under env settings: ENVS="NX_DEC_PAGE=1 NX_DEC_PAGE=0"
for e in $ENVS; do
  for bc in "128 600" "256 600" "64 2000" "4 3000" "16 1000"; do
    set -- $bc
    env $e MODEL=llama3-8b B=$1 CTX=$2 PCTS=${PCTS:-100} REPS=4 timeout 300 python tools/attn_decode_bw.py | sed "s/^{/{\"variant\": \"$e\", /"
  done
done

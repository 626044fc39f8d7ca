# A/B of decode-attention builds (ab/<variant>.so via NX_LIB_PATH) on the attention probe:
# Llama-3.1-8B decode batches on the whole GPU and on a 32-SM lane.
for v in ${VARIANTS:-base p8 p9 p10}; do
  for bc in "128 600" "256 600" "64 2000" "4 3000"; do
    set -- $bc
    NX_LIB_PATH=ab/$v.so MODEL=llama3-8b B=$1 CTX=$2 PCTS=100,21 REPS=4 timeout 300 python tools/attn_decode_bw.py \
      | sed "s/^{/{\"variant\": \"$v\", /"
  done
done

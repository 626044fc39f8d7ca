for sp in 0 1; do
  export NX_GREEN_SPREAD=$sp
  python -c "
from paper_2507_06608_b200 import device as D
d=D.Device(D.arch_preset('tiny') if hasattr(D,'arch_preset') else None)
i=d.info(); print('spread', $sp, 'layouts', i.n_layouts, list(i.layout_decode_sms[:i.n_layouts]), list(i.layout_prefill_sms[:i.n_layouts]))
" 2>&1 | tail -1
  for bc in "128 600" "256 600" "4 3000"; do set -- $bc
    MODEL=llama3-8b B=$1 CTX=$2 PCTS=21,50 REPS=4 python tools/attn_decode_bw.py | sed "s/^{/{\"spread\": $sp, /"
  done
  B=64,128,256 CTX=600 PCTS=21,50 python tools/decode_step_probe.py | sed "s/^{/{\"spread\": $sp, /"
done

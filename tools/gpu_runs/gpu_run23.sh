python - <<'PY'
import re
s=open('bench.py').read()
if '--gamma' not in s:
    s=s.replace('    p.add_argument("--alpha", type=float, default=1.3,', '    p.add_argument("--gamma", type=float, default=15.0, help="ControllerConfig.gamma (SPF aging, tokens/s)")\n    p.add_argument("--alpha", type=float, default=1.3,')
    s=s.replace('    ctrl.alpha, ctrl.beta = alpha, beta', '    ctrl.alpha, ctrl.beta = alpha, beta\n    ctrl.gamma = float(os.environ.get("NX_GAMMA", ctrl.gamma))')
    open('bench.py','w').write(s)
PY
for g in 15 150 1500; do for r in 128 160; do
 NX_GAMMA=$g timeout 900 python bench.py --rate $r --requests 400 --steps 1 --warmup 1 > gpurun_out/g_${g}_${r}.json 2> gpurun_out/g_${g}_${r}.err
done; done

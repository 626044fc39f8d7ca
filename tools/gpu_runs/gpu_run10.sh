timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe.jsonl 2>&1
cat > /tmp/one_o.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2507_06608_b200 import device as D
rng = np.random.default_rng(0)
x = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((64, 4096)).astype(np.float32)))
w = D.Buf.from_array(D.f32_to_bf16(rng.standard_normal((4096, 4096)).astype(np.float32) * 0.02))
o = D.Buf(64 * 4096 * 2)
for _ in range(3): D.gemm(x, w, 64, 4096, 4096, D.EPI_RESIDUAL, o, 4096, residual=o, ldr=4096)
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/gemm_o_streamk python /tmp/one_o.py > /dev/null 2>&1

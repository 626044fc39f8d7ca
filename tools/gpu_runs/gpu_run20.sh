timeout 300 ncu --set full --clock-control none -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/gu_streamk python tools/gemm_case.py > /dev/null 2>&1
SPLITS=2 timeout 300 ncu --set full --clock-control none -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/gu_split2 python tools/gemm_case.py > /dev/null 2>&1
ls gpurun_out

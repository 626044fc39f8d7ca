timeout 600 python -m paper_2507_06608_b200.calibrate --out profiles/b200_llama3_8b > gpurun_out/calib2.json 2> gpurun_out/calib2.err
cp profiles/b200_llama3_8b.* gpurun_out/
for eng in nexus monolithic; do for r in 64 96 128; do
  timeout 600 python bench.py --engine $eng --rate $r --requests 400 --steps 1 --warmup 1 --profile-every 16 --max-decode-batch 128 > gpurun_out/s3_${eng}_${r}.json 2> gpurun_out/s3_${eng}_${r}.err
done; done

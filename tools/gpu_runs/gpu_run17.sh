for beta in 1.1 1.5 2.0 3.0; do for r in 112 128; do
  timeout 600 python bench.py --engine nexus --rate $r --requests 400 --steps 1 --warmup 1 --profile-every 16 --max-decode-batch 128 --beta $beta > gpurun_out/s4_${beta}_${r}.json 2> gpurun_out/s4_${beta}_${r}.err
done; done
timeout 600 python bench.py --engine monolithic --rate 112 --requests 400 --steps 1 --warmup 1 --profile-every 16 --max-decode-batch 128 > gpurun_out/s4_mono_112.json 2> gpurun_out/s4_mono_112.err

mkdir -p gpurun_out
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg"
for mode in "prefill" "decode" "colo"; do
  echo "== $mode"
  RANGE=1 B=96 PPCT=79 DPCT=21 DSTEPS=2 MODE=$mode REPS=3 timeout 600 ncu --replay-mode app-range --clock-control none --metrics $M --csv python tools/step_driver.py > gpurun_out/ay_$mode.csv 2> gpurun_out/ay_$mode.err
  echo "rc $?"; tail -5 gpurun_out/ay_$mode.csv | cut -c1-400
done

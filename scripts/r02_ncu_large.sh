set -x
O=gpurun_out/r02h; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for W in cfg3 cfg4; do
  timeout 300 python scripts/run_once.py $W > $O/plain_$W.log 2>&1; echo plain_$W=$?
  timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_" --csv --log-file $O/metrics_$W.csv python scripts/run_once.py $W > $O/ncu_$W.log 2>&1; echo ncu_$W=$?
done

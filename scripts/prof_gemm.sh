# DMMA pipe utilisation of every large-path contraction GEMM launch of one cfg3 zip-up
# (after the warm-up zip-ups), after a plain run of the same command
C="python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain_cfg3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:k_gemm_dmma -s 600 -c 200 --csv --log-file gpurun_out/gemm_dmma.csv $C > gpurun_out/ncu_gemm.log 2>&1

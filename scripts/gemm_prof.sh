# large-path check: GPU tests of the large-member path, cfg3 bench, and the launch list of one cfg3 zip-up
timeout 900 python -m pytest tests/test_gpu_large.py -x -q -p no:cacheprovider > gpurun_out/pytest_large.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_large.log
C="python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/bench_cfg3.log 2>&1 && ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_gemm|k_qr|k_jacobi|k_mpo|k_copy|k_finish" -s 200 -c 400 --csv --log-file gpurun_out/launches_cfg3.csv $C > gpurun_out/ncu_cfg3.log 2>&1

# round 2, call 5: tall CholeskyQR2 for the a1 sweeps; tests with per-test timeout + durations; cfg3/cfg4 bench
set -x
O=gpurun_out/r02e; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_large.py tests/test_gpu_f32.py tests/test_gpu_variational.py tests/test_gpu_shard.py tests/test_gpu_gemm.py -q -p no:cacheprovider -m "gpu and not slow" --timeout 240 --durations 15 > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -30 $O/pytest.log
for W in cfg3 cfg4 cfg2; do
  timeout 300 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$W.json 2> $O/bench_$W.err; echo $W=$?
done
C="python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/launches_cfg3.csv $C > $O/ncu_cfg3.log 2>&1; echo launches=$?

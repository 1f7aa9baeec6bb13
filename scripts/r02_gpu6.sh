# round 2, call 6: symmetric / triangular GEMM skips + faster Cholesky; large-path tests + bench
set -x
O=gpurun_out/r02f; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_large.py tests/test_gpu_f32.py tests/test_gpu_shard.py tests/test_gpu_variational.py -q -p no:cacheprovider -m "gpu and not slow" --timeout 300 --durations 8 > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -14 $O/pytest.log
for W in cfg3 cfg4 cfg2; do
  timeout 300 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$W.json 2> $O/bench_$W.err; echo $W=$?
done
timeout 300 python bench.py --workload variational --ncores 2 --steps 3 --warmup 3 > $O/bench_var2.json 2> $O/bench_var2.err; echo var2=$?
timeout 300 python bench.py --workload variational --steps 3 --warmup 3 > $O/bench_var1.json 2> $O/bench_var1.err; echo var1=$?
C="python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/launches_cfg3.csv $C > $O/ncu_cfg3.log 2>&1; echo launches=$?

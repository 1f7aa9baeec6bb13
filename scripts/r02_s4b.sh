# session 4: HEAD after the TMA option became a template parameter (libqtt: cp.async feed)
set -x
O=gpurun_out/s4b; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider -s > $O/pytest_gemm.log 2>&1; echo gemm_rc=$?
tail -2 $O/pytest_gemm.log
for W in cfg3 cfg4 cfg2; do timeout 600 python bench.py --workload $W --steps 5 --warmup 3 > $O/bench_$W.json 2> $O/bench_$W.err; echo $W=$?; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?

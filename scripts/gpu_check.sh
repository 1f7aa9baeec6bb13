# quick GPU check: parity tests (minus the 150 s cfg4 full-size case) + default bench
timeout 900 python -m pytest tests -m gpu -x -q -k "not cfg4_full" -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo bench_exit=$? >> gpurun_out/bench.log

set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a/pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r02a/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r02a/bench_cfg5.json 2> gpurun_out/r02a/bench_cfg5.err; echo rc=$?
for w in cfg1 cfg2 cfg4; do timeout 400 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02a/bench_$w.json 2> gpurun_out/r02a/bench_$w.err; echo $w rc=$?; done
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 > gpurun_out/r02a/bench_cfg3.json 2> gpurun_out/r02a/bench_cfg3.err; echo cfg3 rc=$?
timeout 600 python bench.py --workload cfg3 --dtype f32 --steps 5 --warmup 3 > gpurun_out/r02a/bench_cfg3_f32.json 2> gpurun_out/r02a/bench_cfg3_f32.err; echo cfg3f32 rc=$?

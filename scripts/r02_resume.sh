# round 2 re-entry check: full GPU suite on HEAD, smoke, cfg5 + large-path bench lines
set -x
O=gpurun_out/r02resume; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --durations 15 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
for W in cfg2 cfg3 cfg4; do timeout 600 python bench.py --workload $W --steps 5 --warmup 3 > $O/bench_$W.json 2> $O/bench_$W.err; echo $W=$?; done

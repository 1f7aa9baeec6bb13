# round 2, call 7: full GPU suite (incl. slow), smoke, cfg5 bench + e2e + cpu baseline, qft / window lines
set -x
O=gpurun_out/r02g; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --durations 12 > $O/pytest_all.log 2>&1; echo pytest_rc=$?
tail -20 $O/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
timeout 300 python bench.py --workload cfg1 --steps 10 --warmup 3 > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo cfg1=$?
timeout 600 python bench.py --workload cfg3 --dtype f32 --steps 3 --warmup 3 --no-e2e > $O/bench_cfg3_f32.json 2> $O/bench_cfg3_f32.err; echo cfg3f32=$?
timeout 300 python bench.py --workload qft --steps 5 --warmup 3 > $O/bench_qft.json 2> $O/bench_qft.err; echo qft=$?
timeout 600 python bench.py --window 2 --steps 5 --warmup 3 --no-e2e > $O/bench_w2.json 2> $O/bench_w2.err; echo w2=$?

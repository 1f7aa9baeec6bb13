# round 2: tall sites QR first -- parity of the large path, cfg4/cfg3 A/B (QTT_NO_TALLQR=1 = before), cfg4 launch list
set -x
O=gpurun_out/r02tq3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_shard.py tests/test_gpu_f32.py -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -5 $O/pytest.log
for wl in cfg4 cfg3; do
  timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${wl}_tq.json 2> $O/bench_${wl}_tq.err; echo $wl=$?
  QTT_TQ_QR1=1 timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${wl}_old.json 2> $O/bench_${wl}_old.err; echo ${wl}old=$?
done
for f in $O/bench_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('value'), d.get('ms_per_step'))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/launch_cfg4.csv python scripts/run_once.py cfg4 > $O/ncu_cfg4.log 2>&1; echo ncu=$?

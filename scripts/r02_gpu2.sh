# round 2, call 2: new GPU tests, large-path launch lists + ncu of k_qr_coop / k_jacobi_coop, sanitizers
set -x
O=gpurun_out/r02b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_variational.py tests/test_gpu_window.py tests/test_gpu_exact.py -x -q -p no:cacheprovider > $O/pytest_new.log 2>&1; echo pytest_rc=$?
tail -3 $O/pytest_new.log
for W in cfg3 cfg4; do
  C="python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 300 $C > $O/plain_$W.log 2>&1; echo plain_$W=$?
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/launches_$W.csv $C > $O/ncu_$W.log 2>&1; echo launches_$W=$?
done
C="python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_qr_coop|k_jacobi_coop" --launch-skip 24 -c 2 -o $O/large_cfg3 $C > $O/ncu_full_cfg3.log 2>&1; echo full_cfg3=$?
C="python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_qr_coop|k_jacobi_coop" --launch-skip 12 -c 2 -o $O/large_cfg4 $C > $O/ncu_full_cfg4.log 2>&1; echo full_cfg4=$?
for t in racecheck synccheck memcheck; do
  for w in small large window2 var2; do
    timeout 600 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_run.py $w > $O/san_${t}_$w.log 2>&1; echo san_${t}_$w=$?
    tail -2 $O/san_${t}_$w.log
  done
done

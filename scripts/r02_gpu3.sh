# round 2, call 3: f3 two-site + f4 sharded GPU tests; ncu --set full of the main-sweep k_qr_coop / k_jacobi_coop
set -x
O=gpurun_out/r02c; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_variational.py tests/test_gpu_shard.py -x -q -p no:cacheprovider -m "gpu and not slow" > $O/pytest_new.log 2>&1; echo pytest_rc=$?
tail -5 $O/pytest_new.log
C="python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_qr_coop|k_jacobi_coop" --launch-skip 140 -c 2 -o $O/large_cfg3 $C > $O/ncu_full_cfg3.log 2>&1; echo full_cfg3=$?
C="python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_qr_coop|k_jacobi_coop" --launch-skip 58 -c 2 -o $O/large_cfg4 $C > $O/ncu_full_cfg4.log 2>&1; echo full_cfg4=$?

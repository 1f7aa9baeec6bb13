# session 3: A/B of partial Jacobi sweeps (base) against full sweeps (nopart); small-path GPU tests
O=gpurun_out/s3b; mkdir -p $O; rm -f gpurun_out/ab.txt
bash scripts/ab.sh base nopart base nopart > /dev/null 2>&1; cp gpurun_out/ab.txt $O/ab.txt
grep -h -o '"jacobi": {[^}]*}' gpurun_out/ab_base.log gpurun_out/ab_nopart.log > $O/jac.txt
timeout 900 python -m pytest tests/test_gpu_zipup.py tests/test_gpu_large.py tests/test_gpu_exact.py tests/test_gpu_window.py tests/test_gpu_variational.py -m gpu -q -p no:cacheprovider -k "not full_oracle" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log

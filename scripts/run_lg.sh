# large-path tests + one zip-up of each large workload + ncu of the biggest cfg3 Jacobi launch
rm -f gpurun_out/ab.txt
python -m pytest tests/test_gpu_large.py tests/test_gpu_f32.py -q -x > gpurun_out/pt_large.log 2>&1
bash scripts/ab_large.sh cfg3 base
bash scripts/ab_large.sh cfg2 base
bash scripts/ab_large.sh cfg4 base
bash scripts/prof_coopjac.sh

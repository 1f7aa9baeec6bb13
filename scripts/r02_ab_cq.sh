set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_zipup.py tests/test_gpu_window.py tests/test_gpu_large.py tests/test_gpu_variational.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/pt_cq.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pt_cq.log
bash scripts/ab.sh base nocq base nocq
cat gpurun_out/ab.txt

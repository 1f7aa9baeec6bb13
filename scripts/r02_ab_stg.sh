set -x
rm -f gpurun_out/ab.txt
timeout 600 python -m pytest tests/test_gpu_zipup.py tests/test_gpu_large.py::test_cfg5_full_batch_sampled_members -x -q -p no:cacheprovider > gpurun_out/pt_stg.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pt_stg.log
bash scripts/ab.sh base nostg base nostg
cat gpurun_out/ab.txt

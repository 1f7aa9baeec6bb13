# large-path A/B (base = libqtt.so) + large-path / f32 tests
rm -f gpurun_out/ab.txt
python -m pytest tests/test_gpu_large.py tests/test_gpu_f32.py -q -x > gpurun_out/pt_large.log 2>&1
bash scripts/ab_large.sh cfg3 base nb16
bash scripts/ab_large.sh cfg2 base nb16
bash scripts/ab_large.sh cfg4 base

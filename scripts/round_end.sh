# round-end evidence: full GPU suite, default bench (with CPU baseline + e2e), qft bench,
# then the ncu captures of the default bench command (scripts/prof_final.sh)
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1
python bench.py > gpurun_out/bench_final.log 2>&1
python bench.py --workload qft > gpurun_out/bench_qft_final.log 2>&1
bash scripts/prof_final.sh
